// tcgen05.mma throughput microbenchmark (diagnostic, not part of libmec):
// one CTA per SM, one warp issues `iters` x 8 MMAs (M=128, N=n, K=16 bf16,
// both operands from smem, SW128 K-major) into one TMEM accumulator, then
// commits and waits.  Prints cycles per MMA for several N.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_mb tools/mma_microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../paper_1706_06873_b200/csrc/ptx.cuh"

using namespace mec;

// kMode: 0 = SS, elect in asm; 1 = SS, elect block; 2 = TS (A in TMEM cols 256..); 3 = TS + commit per 4
template <int kMode>
__global__ void __launch_bounds__(128, 1) mma_bench(int n, int iters, unsigned long long* cycles, int rnd) {
  constexpr bool kElectInAsm = kMode != 1;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::mbar_init(&bar2, 1);
    ptx::fence_mbar_init();
  }
  // operands: zero, or (rnd) pseudo-random bf16 in about [-1, 1)
  for (int i = threadIdx.x; i < (131072 + 6 * 96 * 128) / 16; i += blockDim.x) {
    uint32_t w[4];
    for (int j = 0; j < 4; ++j) {
      uint32_t x = (i * 4 + j) * 2654435761u + 12345u;
      x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
      // two bf16: sign/exponent around 1.0 (0x3f80), random mantissa and sign
      w[j] = rnd ? (((x & 0x807Fu) | 0x3F00u) | (((x >> 16) & 0x807Fu) | 0x3F00u) << 16) : 0u;
    }
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (warp == 0) ptx::tmem_alloc_dyn(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1) {
    const uint32_t idesc = ptx::instr_desc(false, 128, n);
    const uint64_t ad0 = ptx::smem_desc_sw128(ptx::smem_u32(smem));
    const uint64_t bd0 = ptx::smem_desc_sw128(ptx::smem_u32(smem + (kMode >= 6 ? 131072 : 32768)));
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if constexpr (kMode == 6 || kMode == 7) {
        // kernel-like SS: per "tile" 6 K-atoms of A from a 4-stage ring (2 atoms
        // per stage), B from 6 resident atoms, D rotating over 4 accumulators of
        // n columns, commit per stage (mode 7: D always at column 0)
        const uint32_t d = tmem + (kMode == 6 ? static_cast<uint32_t>((it & 3) * n) : 0u);
#pragma unroll 1
        for (int st = 0; st < 3; ++st) {
          ptx::tc_fence_after();
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const int atom = st * 2 + a;
            const uint64_t ad = ad0 + static_cast<uint32_t>(((it * 3 + st) & 3) * 2048 + a * 1024);
            const uint64_t bd = bd0 + static_cast<uint32_t>(atom * n * 128 / 16);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              ptx::mma_ss_elect<false>(d, ad + 2 * k, bd + 2 * k, idesc, (atom | k) != 0);
          }
          ptx::mma_commit_elect(&bar2);
        }
      } else if constexpr (kMode >= 4) {
        // 7 B atoms (N x 128 B each), 4 MMAs per atom, commit per atom (kernel-like)
#pragma unroll 1
        for (int a = 0; a < 7; ++a) {
          const uint64_t bd = bd0 + static_cast<uint32_t>(a * n * 128 / 16);
          ptx::tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k)
            ptx::mma_ts_elect<false>(tmem, tmem + 256 + 32 * (a & 3) + 8 * k, bd + 2 * k, idesc, (it | a | k) != 0);
          ptx::mma_commit_elect(&bar2);
        }
      } else if constexpr (kMode >= 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          ptx::mma_ts_elect<false>(tmem, tmem + 256 + 8 * (k & 3) + 32 * (k >> 2), bd0 + (k & 3) * 2, idesc,
                                   (it | k) != 0);
          if (kMode == 3 && (k & 3) == 3) ptx::mma_commit_elect(&bar2);
        }
      } else if constexpr (kElectInAsm) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          ptx::mma_ss_elect<false>(tmem, ad0 + (k & 3) * 2 + (k >> 2) * 1024, bd0 + (k & 3) * 2, idesc,
                                   (it | k) != 0);
      } else {
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::mma_ss<false>(tmem, ad0 + (k & 3) * 2 + (k >> 2) * 1024, bd0 + (k & 3) * 2, idesc,
                               (it | k) != 0);
        }
        __syncwarp();
      }
    }
    ptx::mma_commit_elect(&bar);
    ptx::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 32) cycles[blockIdx.x] = t1 - t0;
  }
  if (kMode == 5 && warp >= 2) {
    uint32_t acc = 0;
    const uint32_t base = ptx::smem_u32(smem) + (threadIdx.x & 31) * 24;
    for (int i = 0; i < iters * 40; ++i) {
      const uint2 v = ptx::ld_shared_v2(base + (i & 63) * 8);
      acc += v.x ^ v.y;
    }
    if (acc == 0x12345) cycles[1023] = acc;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

int main(int argc, char** argv) {
  const int rnd = argc > 1 ? atoi(argv[1]) : 0;
  unsigned long long* d;
  cudaMalloc(&d, 1024 * sizeof(unsigned long long));
  const int smem = 131072 + 6 * 96 * 128 + 1024;
  cudaFuncSetAttribute(mma_bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_bench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_bench<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_bench<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_bench<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  const char* names[8] = {"SS elect-in-asm", "SS elect-block ", "TS             ", "TS commit/4    ",
                          "TS 7 B atoms   ", "TS 7B + LDS    ", "SS kernel-like ", "SS kernel D=0  "};
  printf("operands: %s\n", rnd ? "random" : "zero");
  for (int variant = 0; variant < 8; ++variant) {
    for (int n : {32, 64, 96}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (variant == 0) mma_bench<0><<<148, 128, smem>>>(n, iters, d, rnd);
        if (variant == 1) mma_bench<1><<<148, 128, smem>>>(n, iters, d, rnd);
        if (variant == 2) mma_bench<2><<<148, 128, smem>>>(n, iters, d, rnd);
        if (variant == 3) mma_bench<3><<<148, 128, smem>>>(n, iters, d, rnd);
        if (variant == 4) mma_bench<4><<<148, 128, smem>>>(n, iters, d, rnd);
        if (variant == 5) mma_bench<5><<<148, 128, smem>>>(n, iters, d, rnd);
        if (variant == 6) mma_bench<6><<<148, 128, smem>>>(n, iters, d, rnd);
        if (variant == 7) mma_bench<7><<<148, 128, smem>>>(n, iters, d, rnd);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      const double mmas = (variant >= 6 ? 24.0 : (variant >= 4 ? 28.0 : 8.0)) * iters;
      const double flops = 148.0 * mmas * 2.0 * 128 * n * 16;
      printf("%s N=%3d: %.1f cycles/MMA (cta0), %.3f ms, %.0f TFLOP/s  [%s]\n",
             names[variant], n, h[0] / mmas, ms, flops / (ms * 1e-3) / 1e12,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
