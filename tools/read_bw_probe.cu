// read_bw_probe.cu -- DRAM read ceilings on B200 for the A-stream of the sweep
// GEMMs: how fast can the whole chip READ a 2 GB buffer (L2 flushed first) by
//   (a) coalesced LDG.128 (grid-stride, 148 x k CTAs),
//   (b) per-thread 128-byte rows (thread m reads row m's 128 B atom with
//       8 x LDG.128, rows one L-row pitch apart: the sweep copier's pattern),
//   (c) TMA 2-D boxes of 128 rows x 128 B (SW128) into a ring of 16 KB stages,
//       one producer thread per CTA, 1 or 2 CTAs per SM,
//   (d) TMA boxes issued by 2 / 4 producer lanes per CTA.
// Standalone (driver entry point, no libmec).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/read_bw_probe tools/read_bw_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));              \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// (a) coalesced 16-byte loads, `unroll` independent loads per thread per iteration
template <int U>
__global__ void __launch_bounds__(256) ldg_coalesced(const uint4* __restrict__ p, size_t n16, unsigned* out) {
  unsigned acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// (b) the sweep copier pattern: a CTA of 128 threads walks atoms (128 B column
// blocks) of a 128-row tile; thread m loads row m's 128 B (8 x LDG.128).
// Rows are `pitch` bytes apart; tiles are handed out grid-stride.  `A` atoms
// in flight per thread.
template <int A>
__global__ void __launch_bounds__(128) ldg_rows(const unsigned char* __restrict__ base, size_t pitch, int n_tiles,
                                                int atoms_per_row, unsigned* out) {
  unsigned acc = 0;
  // work unit = (tile, chunk of atoms_per_row atoms); units grid-stride
  const int chunks = static_cast<int>(pitch / 128) / atoms_per_row;
  for (int w = blockIdx.x; w < n_tiles * chunks; w += gridDim.x) {
    const int t = w / chunks;
    const unsigned char* row = base + (static_cast<size_t>(t) * 128 + threadIdx.x) * pitch +
                               static_cast<size_t>(w % chunks) * atoms_per_row * 128;
    for (int a = 0; a + A <= atoms_per_row; a += A) {
      uint4 v[A][8];
#pragma unroll
      for (int u = 0; u < A; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) v[u][k] = __ldcs(reinterpret_cast<const uint4*>(row + (a + u) * 128) + k);
#pragma unroll
      for (int u = 0; u < A; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[u][k].x ^ v[u][k].w;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// (c)/(d) TMA boxes of 128 rows x 128 B into `stages` 16 KB stages per producer
// lane; `lanes` producer lanes of warp 0, each with its own ring.  A tile's
// atoms are walked in order (x = atom * 64 elements), tiles grid-stride.
__global__ void __launch_bounds__(128) tma_rows(const __grid_constant__ CUtensorMap tm, int n_tiles,
                                                int atoms_per_row, int stages, int lanes, int chunks,
                                                unsigned char* wbuf = nullptr, size_t wbytes_per_unit = 0) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[32];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 32; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int lane = threadIdx.x;
  if (wbuf != nullptr && threadIdx.x >= 32) {
    // (e) warps 1-3 write wbytes_per_unit bytes per work unit to a disjoint
    // buffer with 16-byte streaming stores (a read/write mix like the GEMM's)
    const int t = threadIdx.x - 32;
    for (int w = blockIdx.x; w < n_tiles * chunks; w += gridDim.x) {
      uint4* dst = reinterpret_cast<uint4*>(wbuf + static_cast<size_t>(w) * wbytes_per_unit);
      for (size_t i = t; i < wbytes_per_unit / 16; i += 96) __stcs(dst + i, make_uint4(w, i, 0, 0));
    }
    return;
  }
  if (lane >= lanes) return;
  uint32_t phase_bits = 0;
  int issued = 0;
  // lane l takes atoms l, l + lanes, ... of the CTA's sequence
  for (int w = blockIdx.x; w < n_tiles * chunks; w += gridDim.x) {
    const int t = w / chunks, a0 = (w % chunks) * atoms_per_row;
    for (int a = a0 + lane; a < a0 + atoms_per_row; a += lanes) {
      const int s = issued % stages;
      if (issued >= stages) {
        const uint32_t par = (phase_bits >> s) & 1u;
        asm volatile(
            "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                su32(&full[lane * stages + s])),
            "r"(par));
        phase_bits ^= 1u << s;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[lane * stages + s])),
                   "r"(16384));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
          "[%4];" ::"r"(su32(smem + (lane * stages + s) * 16384)),
          "l"(&tm), "r"(a * 64), "r"(t * 128), "r"(su32(&full[lane * stages + s]))
          : "memory");
      ++issued;
    }
  }
  for (int k = issued > stages ? issued - stages : 0; k < issued; ++k) {
    const int s = k % stages;
    const uint32_t par = (phase_bits >> s) & 1u;
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                     su32(&full[lane * stages + s])),
                 "r"(par));
    phase_bits ^= 1u << s;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  // L-like buffer: rows of 43008 bf16 (C2's L row, 86 KB), 24576 rows = 2.1 GB
  const size_t cols = 43008, rows = 24576, pitch = cols * 2, bytes = pitch * rows;
  unsigned char* src = nullptr;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 1, bytes));
  void* flush = nullptr;
  CK(cudaMalloc(&flush, 512u << 20));
  unsigned* out = nullptr;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timed = [&](auto launch) -> float {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(flush, r, 512u << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best;
  };
  const size_t n16 = bytes / 16;
  for (int ctas_per_sm : {4, 8}) {
    float ms = timed([&] { ldg_coalesced<4><<<sms * ctas_per_sm, 256>>>(reinterpret_cast<const uint4*>(src), n16, out); });
    printf("(a) LDG.128 coalesced, %d x 256 thr/SM, 4 in flight: %.1f us, %.0f GB/s\n", ctas_per_sm, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9);
    ms = timed([&] { ldg_coalesced<8><<<sms * ctas_per_sm, 256>>>(reinterpret_cast<const uint4*>(src), n16, out); });
    printf("(a) LDG.128 coalesced, %d x 256 thr/SM, 8 in flight: %.1f us, %.0f GB/s\n", ctas_per_sm, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9);
  }
  // (b) the sweep pattern reads atoms_per_row atoms of every row (whole rows here)
  // 672 atoms per row = 7 chunks of 96 atoms (a sweep item's stream length): 1344 units
  const int n_tiles = static_cast<int>(rows / 128), apr = 96, chunks = static_cast<int>(pitch / 128) / apr;
  for (int ctas_per_sm : {1, 2, 4, 8}) {
    float ms = timed([&] { ldg_rows<1><<<sms * ctas_per_sm, 128>>>(src, pitch, n_tiles, apr, out); });
    printf("(b) LDG rows, %d CTAs/SM, 1 atom in flight/thread: %.1f us, %.0f GB/s\n", ctas_per_sm, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9);
    ms = timed([&] { ldg_rows<2><<<sms * ctas_per_sm, 128>>>(src, pitch, n_tiles, apr, out); });
    printf("(b) LDG rows, %d CTAs/SM, 2 atoms in flight/thread: %.1f us, %.0f GB/s\n", ctas_per_sm, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9);
    ms = timed([&] { ldg_rows<4><<<sms * ctas_per_sm, 128>>>(src, pitch, n_tiles, apr, out); });
    printf("(b) LDG rows, %d CTAs/SM, 4 atoms in flight/thread: %.1f us, %.0f GB/s\n", ctas_per_sm, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9);
  }
  CUtensorMap tm;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {pitch};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  CK(cudaFuncSetAttribute(tma_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384));
  for (int ctas_per_sm : {1, 2}) {
    for (int lanes : {1, 2, 4}) {
      for (int stages : {4, 6, 12}) {
        if (lanes * stages > 12 || (ctas_per_sm == 2 && lanes * stages > 6)) continue;
        float ms = timed([&] {
          tma_rows<<<sms * ctas_per_sm, 128, lanes * stages * 16384>>>(tm, n_tiles, apr, stages, lanes, chunks);
        });
        printf("(c) TMA 128x128B boxes, %d CTA/SM, %d lanes x %d stages: %.1f us, %.0f GB/s\n", ctas_per_sm, lanes,
               stages, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
      }
    }
  }
  // (e) TMA reads + 16-byte stores at the C2 GEMM's mix (O / L = 0.33)
  unsigned char* wbuf = nullptr;
  const size_t wpu = static_cast<size_t>(apr) * 16384 / 3;  // per unit: a third of its read bytes
  CK(cudaMalloc(&wbuf, wpu * n_tiles * chunks + 4096));
  for (int stages : {6, 12}) {
    float ms = timed([&] {
      tma_rows<<<sms, 128, stages * 16384>>>(tm, n_tiles, apr, stages, 1, chunks, wbuf, wpu);
    });
    const double tot = bytes + static_cast<double>(wpu) * n_tiles * chunks;
    printf("(e) TMA reads + st.global writes (1/3), %d stages: %.1f us, %.0f GB/s total (%.0f read)\n", stages,
           ms * 1e3, tot / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
