// format_fix.cu -- Solution A's paper-literal format fix (Alg.2 l.13-19,
// P:173-183), used with MEC_SOLA_FIX_LITERAL:
//   l.13      Copy L = O                      (O holds h-n-w-c after l.10-12)
//   l.14-19   O[n, h, 0:o_w k_c] = L[h, n, 0:o_w k_c]
// Pure data movement (HBM-bound): 128-bit loads/stores when the block size
// o_w k_c elt is a multiple of 16 bytes, element copies otherwise.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mec_internal.h"

namespace mec {
namespace {

__global__ void __launch_bounds__(256) copy16_kernel(const uint4* __restrict__ src,
                                                     uint4* __restrict__ dst, int64_t n16,
                                                     const unsigned char* __restrict__ src_b,
                                                     unsigned char* __restrict__ dst_b,
                                                     int64_t tail_from, int64_t nbytes) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += stride)
    dst[i] = src[i];
  for (int64_t b = tail_from + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       b < nbytes; b += stride)
    dst_b[b] = src_b[b];
}

// One CTA per destination block (n, h): O[(n o_h + h) blk] = L[(h i_n + n) blk].
__global__ void __launch_bounds__(256) block_permute_kernel(const unsigned char* __restrict__ L,
                                                            unsigned char* __restrict__ O,
                                                            int64_t i_n, int64_t o_h,
                                                            int64_t blk_bytes, bool vec) {
  const int64_t b = blockIdx.x;  // destination block index n o_h + h
  const int64_t n = b / o_h, h = b - n * o_h;
  const unsigned char* src = L + (h * i_n + n) * blk_bytes;
  unsigned char* dst = O + b * blk_bytes;
  if (vec) {
    const int64_t n16 = blk_bytes / 16;
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  } else {
    for (int64_t i = threadIdx.x; i < blk_bytes; i += blockDim.x) dst[i] = src[i];
  }
}

}  // namespace

cudaError_t launch_sola_copy(const Plan& p, const void* O, void* Laux, cudaStream_t st,
                             int* launches) {
  const int64_t nbytes = p.n_O * p.elt;
  const int64_t n16 = nbytes / 16;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((n16 + 255) / 256, 8LL * num_sms()));
  copy16_kernel<<<static_cast<unsigned>(grid), 256, 0, st>>>(
      static_cast<const uint4*>(O), static_cast<uint4*>(Laux), n16,
      static_cast<const unsigned char*>(O), static_cast<unsigned char*>(Laux), n16 * 16, nbytes);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_sola_transpose(const Plan& p, const void* Laux, void* O, cudaStream_t st,
                                  int* launches) {
  const int64_t blk_bytes = p.o_w * p.s.k_c * p.elt;
  const int64_t nblk = p.s.i_n * p.o_h;
  if (nblk > 0x7FFFFFFF) return cudaErrorInvalidConfiguration;
  block_permute_kernel<<<static_cast<unsigned>(nblk), 256, 0, st>>>(
      static_cast<const unsigned char*>(Laux), static_cast<unsigned char*>(O), p.s.i_n, p.o_h,
      blk_bytes, blk_bytes % 16 == 0);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace mec
