// tcgen05.mma throughput microbenchmark (diagnostic, not part of libmec):
// one CTA per SM, one warp issues `iters` x 8 MMAs (M=128, N=n, K=16 bf16,
// both operands from smem, SW128 K-major) into one TMEM accumulator, then
// commits and waits.  Prints cycles per MMA for several N.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_mb tools/mma_microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_1706_06873_b200/csrc/ptx.cuh"

using namespace mec;

template <bool kElectInAsm>
__global__ void __launch_bounds__(128, 1) mma_bench(int n, int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  // zero operands
  for (int i = threadIdx.x; i < (32768 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) ptx::tmem_alloc_dyn(&tslot, 256);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1) {
    const uint32_t idesc = ptx::instr_desc(false, 128, n);
    const uint64_t ad0 = ptx::smem_desc_sw128(ptx::smem_u32(smem));
    const uint64_t bd0 = ptx::smem_desc_sw128(ptx::smem_u32(smem + 32768));
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if constexpr (kElectInAsm) {
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
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * sizeof(unsigned long long));
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(mma_bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  for (int variant = 0; variant < 2; ++variant) {
    for (int n : {32, 64, 96, 128, 192, 256}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (variant == 0)
          mma_bench<true><<<148, 128, smem>>>(n, iters, d);
        else
          mma_bench<false><<<148, 128, smem>>>(n, iters, d);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      const double mmas = 8.0 * iters;
      const double flops = 148.0 * mmas * 2.0 * 128 * n * 16;
      printf("%s N=%3d: %.1f cycles/MMA (cta0), %.3f ms, %.0f TFLOP/s  [%s]\n",
             variant == 0 ? "elect-in-asm" : "elect-block ", n, h[0] / mmas, ms, flops / (ms * 1e-3) / 1e12,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
