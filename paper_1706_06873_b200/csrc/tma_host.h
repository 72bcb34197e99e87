// tma_host.h -- host-side TMA tensor-map encoding through the driver entry
// point (no link-time dependency on libcuda; the runtime resolves it).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace mec {

// Tiled tensor map, 128-byte swizzle, zero OOB fill, 256-byte L2 promotion.
// Element type BFLOAT16 (tf32 == false) or FLOAT32 (tf32 == true; the tensor
// core reads fp32 storage as tf32).  Returns cudaErrorInvalidValue if the
// driver rejects the parameters.
cudaError_t encode_tiled(CUtensorMap* map, bool tf32, int rank, const void* base,
                         const uint64_t* dims, const uint64_t* strides_bytes,
                         const uint32_t* box);

// Same with an explicit swizzle span in bytes (0 = none, 32, 64, 128), for
// the epilogue's TMA stores.
cudaError_t encode_tiled_swz(CUtensorMap* map, bool tf32, int rank, const void* base,
                             const uint64_t* dims, const uint64_t* strides_bytes,
                             const uint32_t* box, int swizzle_bytes);

// Tiled map with per-dimension traversal strides (elementStrides), 128-byte
// swizzle: the fused path's view of the NHWC input (pixel stride s_w).
cudaError_t encode_tiled_strided(CUtensorMap* map, bool tf32, int rank, const void* base,
                                 const uint64_t* dims, const uint64_t* strides_bytes,
                                 const uint32_t* box, const uint32_t* elem_strides);

}  // namespace mec
