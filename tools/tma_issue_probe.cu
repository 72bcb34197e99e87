// tma_issue_probe.cu -- how fast can one thread per SM stream 16 KB TMA boxes
// (the sweep GEMM's A atoms) into a ring of shared-memory stages?  Measures the
// cycles a TMA issue blocks the issuing thread and the sustained bytes/s per SM
// and chip, for boxes of 128 rows x 128 B (one per atom) and 2 x 64 rows,
// with the source resident in L2 or not.  Standalone (driver entry point, no
// libmec).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/tma_issue_probe tools/tma_issue_probe.cu     Run: tools/tma_issue_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));              \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tm, int rows_box, int n_atoms,
                                                int stages, int row_step, long long* out_issue, long long* out_total,
                                                const void* bulk_src) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[32];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int boxes = rows_box > 0 ? 128 / rows_box : (rows_box == 0 ? 1 : -rows_box);
  const unsigned char* gsrc = reinterpret_cast<const unsigned char*>(bulk_src);
  long long t_issue = 0;
  const long long t0 = clock64();
  uint32_t phase_bits = 0;
  for (int a = 0; a < n_atoms; ++a) {
    const int s = a % stages;
    if (a >= stages) {  // the stage's previous load must have landed
      const uint32_t par = (phase_bits >> s) & 1u;
      asm volatile(
          "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
              su32(&full[s])),
          "r"(par));
      phase_bits ^= 1u << s;
    }
    const long long c0 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(16384));
    for (int b = 0; b < boxes && rows_box <= 0; ++b) {  // 1-D bulk copies of contiguous bytes
      const uint32_t chunk = 16384u / static_cast<uint32_t>(boxes);
      const size_t off = (static_cast<size_t>(blockIdx.x) * row_step * 8192 + static_cast<size_t>(a % 64) * 16384 +
                          static_cast<size_t>(a / 64) * 64 * 16384 + b * chunk) %
                         (static_cast<size_t>(512) << 20);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              su32(smem + s * 16384 + b * chunk)),
          "l"(gsrc + off), "r"(chunk), "r"(su32(&full[s]))
          : "memory");
    }
    for (int b = 0; b < boxes && rows_box > 0; ++b) {
      const int x = (a % 64) * 64;
      const int y = (blockIdx.x * row_step + (a / 64) * 128 + b * rows_box) % 65536;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(smem + s * 16384 + b * rows_box * 128)),
          "l"(&tm), "r"(x), "r"(y), "r"(su32(&full[s]))
          : "memory");
    }
    t_issue += clock64() - c0;
  }
  for (int a = n_atoms > stages ? n_atoms - stages : 0; a < n_atoms; ++a) {
    const int s = a % stages;
    const uint32_t par = (phase_bits >> s) & 1u;
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                     su32(&full[s])),
                 "r"(par));
    phase_bits ^= 1u << s;
  }
  out_issue[blockIdx.x] = t_issue;
  out_total[blockIdx.x] = clock64() - t0;
}


// nw producer warps in one CTA, each streaming its own ring of `stages` 16 KB stages
__global__ void __launch_bounds__(128, 1) probe_warps(const __grid_constant__ CUtensorMap tm, int nw, int n_atoms,
                                                      int stages, int lanes, long long* out_total, int disjoint) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 32; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long long t0 = clock64();
  if (warp < nw && lane < lanes) {
    // ring r = (warp, lane): stages [r stages, (r + 1) stages)
    const int r = warp * lanes + lane;
    uint32_t phase_bits = 0;
    for (int a = 0; a < n_atoms; ++a) {
      const int s = r * stages + a % stages;
      if (a >= stages) {
        const uint32_t par = (phase_bits >> (a % stages)) & 1u;
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                         su32(&full[s])), "r"(par));
        phase_bits ^= 1u << (a % stages);
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(16384));
      const int x = (a % 64) * 64;
      const int y = ((a / 64) * 128 + r * 512 + (disjoint ? blockIdx.x * 2048 : 0)) % 65536;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(smem + s * 16384)), "l"(&tm), "r"(x), "r"(y), "r"(su32(&full[s])) : "memory");
    }
    for (int a = n_atoms > stages ? n_atoms - stages : 0; a < n_atoms; ++a) {
      const int s = r * stages + a % stages;
      const uint32_t par = (phase_bits >> (a % stages)) & 1u;
      asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                       su32(&full[s])), "r"(par));
      phase_bits ^= 1u << (a % stages);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out_total[blockIdx.x] = clock64() - t0;
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
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  // source: 65536 rows x 4096 bf16 (8 KB) = 512 MB; the kernel touches a window
  const size_t cols = 4096, rows = 65536;
  void* src = nullptr;
  CK(cudaMalloc(&src, cols * rows * 2));
  CK(cudaMemset(src, 1, cols * rows * 2));
  void* flush = nullptr;
  CK(cudaMalloc(&flush, 512u << 20));
  long long *d_issue, *d_total;
  CK(cudaMalloc(&d_issue, sizeof(long long) * 1024));
  CK(cudaMalloc(&d_total, sizeof(long long) * 1024));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 13 * 16384));
  for (int rows_box : {128, 64, 32, 0, -4}) {
    CUtensorMap tm;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(rows_box > 0 ? rows_box : 128)};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    for (int ctas : {1, sms}) {
      for (int l2 : {0, 1}) {
        const int n_atoms = 256, stages = 8;
        // L2-resident: every CTA reads the same 4 MB window (row_step 0) after a warm-up run;
        // DRAM: disjoint windows (row_step 256 rows) after a flush
        const int row_step = l2 ? 0 : 256;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        if (l2) probe<<<ctas, 128, stages * 16384>>>(tm, rows_box, n_atoms, stages, row_step, d_issue, d_total, src);
        else CK(cudaMemset(flush, 0, 512u << 20));
        CK(cudaEventRecord(e0));
        probe<<<ctas, 128, stages * 16384>>>(tm, rows_box, n_atoms, stages, row_step, d_issue, d_total, src);
        CK(cudaEventRecord(e1));
        CK(cudaDeviceSynchronize());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        std::vector<long long> iss(ctas), tot(ctas);
        CK(cudaMemcpy(iss.data(), d_issue, sizeof(long long) * ctas, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(tot.data(), d_total, sizeof(long long) * ctas, cudaMemcpyDeviceToHost));
        std::sort(iss.begin(), iss.end());
        std::sort(tot.begin(), tot.end());
        const double bytes = 16384.0 * n_atoms;
        const double cyc = static_cast<double>(tot[ctas / 2]);
        printf("box %3d rows x 128 B (%d per atom), CTAs %3d, %s: issue %.0f cyc/atom (median CTA), in-kernel %.0f "
               "cyc/atom = %.1f GB/s per SM; event %.1f us -> %.0f GB/s chip\n",
               rows_box, rows_box > 0 ? 128 / rows_box : (rows_box == 0 ? 1 : -rows_box), ctas, l2 ? "L2-resident" : "after flush", iss[ctas / 2] / double(n_atoms),
               cyc / n_atoms, bytes / (cyc / (clk * 1e3)) / 1e9, ms * 1e3, bytes * ctas / (ms * 1e-3) / 1e9);
      }
    }
  }
  {  // stages in flight, one or two CTAs per SM, 128-row boxes, L2-resident
    CUtensorMap tm;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int per_sm : {1, 2})
      for (int stages : {2, 4, 6, 8, 12}) {
        if (per_sm * stages * 16384 > 220 * 1024) continue;
        const int ctas = per_sm * sms, n_atoms = 256;
        probe<<<ctas, 128, stages * 16384>>>(tm, 128, n_atoms, stages, 0, d_issue, d_total, src);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0));
        probe<<<ctas, 128, stages * 16384>>>(tm, 128, n_atoms, stages, 0, d_issue, d_total, src);
        CK(cudaEventRecord(e1));
        CK(cudaDeviceSynchronize());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("L2-resident, %d CTA(s) per SM, %2d stages of 16 KB: %.1f GB/s per SM, %.0f GB/s chip\n", per_sm, stages,
               16384.0 * n_atoms * per_sm / (ms * 1e-3) / 1e9, 16384.0 * n_atoms * ctas / (ms * 1e-3) / 1e9);
      }
  }
  {  // producer warps / lanes per CTA, one CTA per SM
    CUtensorMap tm;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CK(cudaFuncSetAttribute(probe_warps, cudaFuncAttributeMaxDynamicSharedMemorySize, 13 * 16384));
    struct Cfg { int nw, lanes, stages; };
    for (Cfg c : {Cfg{1, 1, 8}, Cfg{2, 1, 4}, Cfg{4, 1, 3}, Cfg{1, 2, 4}, Cfg{1, 4, 3}}) {
      for (int l2 : {1, 0}) {
        const int n_atoms = 256;
        if (l2) probe_warps<<<sms, 128, 13 * 16384>>>(tm, c.nw, n_atoms, c.stages, c.lanes, d_total, 1 - l2);
        else CK(cudaMemset(flush, 0, 512u << 20));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0));
        probe_warps<<<sms, 128, 13 * 16384>>>(tm, c.nw, n_atoms, c.stages, c.lanes, d_total, 1 - l2);
        CK(cudaEventRecord(e1));
        CK(cudaDeviceSynchronize());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double b = 16384.0 * n_atoms * c.nw * c.lanes;
        printf("%s: %d producer warp(s) x %d lane(s), %d stages each: %.1f GB/s per SM, %.0f GB/s chip\n",
               l2 ? "L2-resident (same windows in every CTA)" : "after flush, disjoint windows (DRAM)", c.nw, c.lanes, c.stages,
               b / (ms * 1e-3) / 1e9, b * sms / (ms * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
