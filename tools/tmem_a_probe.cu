// Probe (diagnostic, not part of libmec): can a tcgen05.mma take its A
// operand from TMEM at ANY 32-bit column (2 bf16 elements), and does
// tcgen05.cp.128x256b copy a 32-byte K chunk of a TMA-style SW128 smem atom
// into TMEM with row m -> lane m?  Both decide whether the window GEMM can
// stream the union of R output rows' windows once and address each row's
// window at its exact element offset (AlexNet conv1: shift 132 bf16 = 66
// columns).  Also times TS MMAs (N = 96) at aligned / unaligned A columns.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_a_probe tools/tmem_a_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_1706_06873_b200/csrc/ptx.cuh"

using namespace mec;

__host__ __device__ inline float a_val(int m, int e) { return static_cast<float>(((m * 7 + e * 3) % 17) - 8); }
__host__ __device__ inline float b_val(int n, int k) { return static_cast<float>(((n * 5 + k * 11) % 13) - 6); }

__device__ inline uint16_t bf16_bits(float f) {  // exact for small integers
  return static_cast<uint16_t>(__float_as_uint(f) >> 16);
}

__device__ inline void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

constexpr int kOffs = 12;
__constant__ int c_offs[kOffs] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 10, 66, 130};

// out_mma[o][m][n] (n < 32); out_cp[m][j] (j < 32 columns); cyc[2]
__global__ void __launch_bounds__(128, 1) probe(float* out_mma, uint32_t* out_cp, float* out_cpmma,
                                                 unsigned long long* cyc, int mode, int the_off) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = threadIdx.x;  // TMEM lane of this thread (warp w -> lanes 32w..)
  unsigned char* atomA = smem;            // 128 rows x 128 B, SW128 (16 KB)
  unsigned char* atomB = smem + 16384;    // 96 rows x 128 B, SW128 (12 KB)
  // fill A atom (elements 0..63 of A row m) and B (n < 96, k < 64), swizzled
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    const uint32_t off = r * 128 + ((((k * 2) >> 4) ^ (r & 7)) << 4) + ((k * 2) & 15);
    *reinterpret_cast<uint16_t*>(atomA + off) = bf16_bits(a_val(r, k));
    if (r < 96) *reinterpret_cast<uint16_t*>(atomB + off) = bf16_bits(b_val(r, k));
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc_dyn(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t lane_base = static_cast<uint32_t>(32 * warp) << 16;
  // A_full[m][0:512] into TMEM columns 256..511 (column j: elements 2j, 2j+1)
  for (int c0 = 0; c0 < 256; c0 += 32) {
    uint32_t r[32];
    for (int j = 0; j < 32; ++j) {
      const int e = 2 * (c0 + j);
      r[j] = static_cast<uint32_t>(bf16_bits(a_val(m, e))) | (static_cast<uint32_t>(bf16_bits(a_val(m, e + 1))) << 16);
    }
    ptx::tmem_st_32x32b_x32(tmem + lane_base + 256 + c0, r);
  }
  ptx::tmem_st_wait();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint64_t bdesc = ptx::smem_desc_sw128(ptx::smem_u32(atomB));
  uint32_t ph = 0;
  for (int o = 0; o < kOffs && mode == 0; ++o) {
    if (c_offs[o] != the_off) continue;
    if (warp == 0) {
      ptx::mma_ts_elect<false>(tmem + 0, tmem + 256 + c_offs[o], bdesc, ptx::instr_desc(false, 128, 32), 0u);
      ptx::mma_commit_elect(&bar);
    }
    ptx::mbar_wait(&bar, ph);
    ph ^= 1;
    ptx::tc_fence_after();
    uint32_t v[16];
    for (int h = 0; h < 2; ++h) {
      ptx::tmem_ld_32x32b_x16(tmem + lane_base + 16 * h, v);
      ptx::tmem_ld_wait();
      for (int j = 0; j < 16; ++j) out_mma[(o * 128 + m) * 32 + 16 * h + j] = __uint_as_float(v[j]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  }
  // tcgen05.cp: the 4 32-byte K chunks of the SW128 A atom -> TMEM columns 128 + 8k
  if (mode == 1 && warp == 0) {
    if (lane == 0) {
      const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(atomA));
      for (int k = 0; k < 4; ++k) tmem_cp_128x256b(tmem + 128 + 8 * k, ad + 2 * k);
      // and an MMA reading the copied A at column offset 2 (elements 4..19);
      // the_off = 1: at column 0 instead (the 4-column rule: offsets 1-3 trap)
      asm volatile(
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 0;" ::"r"(tmem + 64),
          "r"(tmem + (the_off == 1 ? 128 : 130)), "l"(bdesc), "r"(ptx::instr_desc(false, 128, 32))
          : "memory");
      ptx::mma_commit(&bar);
    }
    __syncwarp();
  }
  if (mode == 1) {
  ptx::mbar_wait(&bar, ph);
  ph ^= 1;
  ptx::tc_fence_after();
  }
  if (mode == 1) {
    uint32_t v[16];
    for (int h = 0; h < 2; ++h) {
      ptx::tmem_ld_32x32b_x16(tmem + lane_base + 128 + 16 * h, v);
      ptx::tmem_ld_wait();
      for (int j = 0; j < 16; ++j) out_cp[m * 32 + 16 * h + j] = v[j];
      ptx::tmem_ld_32x32b_x16(tmem + lane_base + 64 + 16 * h, v);
      ptx::tmem_ld_wait();
      for (int j = 0; j < 16; ++j) out_cpmma[m * 32 + 16 * h + j] = __uint_as_float(v[j]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // timing: 2048 TS MMAs N=96 at A column 256 + 8k (aligned) vs 256 + 2 + 8k
  for (int t = 0; t < 2 && (mode == 2 || mode == 3); ++t) {
    if (mode == 2 && t == 1) break;
    if (mode == 3 && t == 0) continue;
    if (warp == 0) {
      const uint32_t idesc = ptx::instr_desc(false, 128, 96);
      const long long t0 = clock64();
      for (int it = 0; it < 512; ++it)
        ptx::mma_ts_atom_elect<false>(tmem + 0, tmem + 256 + (t ? 2 : 0) + 32 * (it & 3), bdesc, idesc, 1u);
      ptx::mma_commit_elect(&bar);
      ptx::mbar_wait(&bar, ph);
      if (lane == 0) cyc[t] = clock64() - t0;
    } else {
      ptx::mbar_wait(&bar, ph);
    }
    ph ^= 1;
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  }
  // sweep-like pattern: rows of 36 TS MMAs (9 groups of 4) alternating two
  // accumulators of N = the_off columns, A at 8-column steps in cols 256..
  if (mode == 5 || mode == 6) {
    if (warp == 0) {
      const uint32_t n = static_cast<uint32_t>(the_off);
      const uint32_t idesc = ptx::instr_desc(false, 128, n);
      const long long t0 = clock64();
      for (int r = 0; r < 64; ++r) {
        const uint32_t d = tmem + static_cast<uint32_t>((r & 1) * n);
        for (int g = 0; g < 9; ++g) {
          const uint32_t col = tmem + 256 + static_cast<uint32_t>(((r * 3 + g) % 7) * 32 + (mode == 6 ? 8 : 0));
          ptx::mma_ts_atom_elect<false>(d, col, bdesc, idesc, g != 0 ? 1u : 0u);
        }
      }
      ptx::mma_commit_elect(&bar);
      ptx::mbar_wait(&bar, ph);
      if (lane == 0) cyc[0] = clock64() - t0;
    } else {
      ptx::mbar_wait(&bar, ph);
    }
    ph ^= 1;
  }
  // mode 7 / 8: tcgen05.cp from a NON-swizzled K-major atom laid out as
  // [16-byte K chunk c][row m][16 B] (8x16 B core matrices contiguous: SBO =
  // 128 B between 8-row groups, LBO = 2048 B between K chunks), copy k takes
  // chunks 2k, 2k+1 (start + 4096 k) -> TMEM columns 128 + 8k; then an MMA on
  // the copied A (columns 128.., K elements 0..15).  Mode 8: throughput.
  if (mode == 7 || mode == 8) {
    unsigned char* atomN = smem + 16384 + 12288;  // 16 KB
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
      const int r = i / 64, k = i % 64;
      *reinterpret_cast<uint16_t*>(atomN + (k / 8) * 2048 + r * 16 + (k % 8) * 2) = bf16_bits(a_val(r, k));
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (warp == 0 && lane == 0) {
      auto ndesc = [&](uint32_t addr) {
        uint64_t d = 0;
        d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
        d |= static_cast<uint64_t>(2048 >> 4) << 16;  // LBO: next K core-matrix column
        d |= static_cast<uint64_t>(128 >> 4) << 32;   // SBO: next 8-row group
        d |= static_cast<uint64_t>(1) << 46;          // version
        return d;                                     // layout 0 = no swizzle
      };
      const uint32_t base = ptx::smem_u32(atomN);
      const long long t0 = clock64();
      const int reps = mode == 8 ? 256 : 1;
      for (int it = 0; it < reps; ++it)
        for (int k = 0; k < 4; ++k) tmem_cp_128x256b(tmem + 128 + 8 * k, ndesc(base + 4096 * k));
      if (mode == 7)
        asm volatile(
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 0;" ::"r"(tmem + 64),
            "r"(tmem + 128), "l"(bdesc), "r"(ptx::instr_desc(false, 128, 32))
            : "memory");
      ptx::mma_commit(&bar);
      ptx::mbar_wait(&bar, ph);
      cyc[2] = clock64() - t0;
    }
    __syncwarp();
    ptx::mbar_wait(&bar, ph);
    ph ^= 1;
    ptx::tc_fence_after();
    if (mode == 7) {
      uint32_t v[16];
      for (int h = 0; h < 2; ++h) {
        ptx::tmem_ld_32x32b_x16(tmem + lane_base + 128 + 16 * h, v);
        ptx::tmem_ld_wait();
        for (int j = 0; j < 16; ++j) out_cp[m * 32 + 16 * h + j] = v[j];
        ptx::tmem_ld_32x32b_x16(tmem + lane_base + 64 + 16 * h, v);
        ptx::tmem_ld_wait();
        for (int j = 0; j < 16; ++j) out_cpmma[m * 32 + 16 * h + j] = __uint_as_float(v[j]);
      }
    }
  }
  // tcgen05.cp throughput: 1024 copies of 128x256b (4 KB each)
  if (mode == 4 && warp == 0) {
    const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(atomA));
    const long long t0 = clock64();
    if (lane == 0) {
      for (int it = 0; it < 1024; ++it) tmem_cp_128x256b(tmem + 128 + 8 * (it & 15), ad + 2 * (it & 3));
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    ptx::mbar_wait(&bar, ph);
    if (lane == 0) cyc[2] = clock64() - t0;
  } else if (mode == 4) {
    ptx::mbar_wait(&bar, ph);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

static float bf(float x) { return x; }

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0, the_off = argc > 2 ? atoi(argv[2]) : 0;
  float *d_mma, *d_cpmma;
  uint32_t* d_cp;
  unsigned long long* d_cyc;
  cudaMalloc(&d_mma, kOffs * 128 * 32 * 4);
  cudaMalloc(&d_cp, 128 * 32 * 4);
  cudaMalloc(&d_cpmma, 128 * 32 * 4);
  cudaMalloc(&d_cyc, 3 * 8);
  const int smem = 16384 + 12288 + 16384 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemset(d_mma, 0xff, kOffs * 128 * 32 * 4);
  probe<<<1, 128, smem>>>(d_mma, d_cp, d_cpmma, d_cyc, mode, the_off);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  static float h_mma[kOffs * 128 * 32], h_cpmma[128 * 32];
  static uint32_t h_cp[128 * 32];
  unsigned long long cyc[3];
  cudaMemcpy(h_mma, d_mma, sizeof(h_mma), cudaMemcpyDeviceToHost);
  cudaMemcpy(h_cp, d_cp, sizeof(h_cp), cudaMemcpyDeviceToHost);
  cudaMemcpy(h_cpmma, d_cpmma, sizeof(h_cpmma), cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  const int offs[kOffs] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 10, 66, 130};
  for (int o = 0; o < kOffs && mode == 0; ++o) {
    if (offs[o] != the_off) continue;
    int bad = 0;
    for (int mm = 0; mm < 128; ++mm)
      for (int n = 0; n < 32; ++n) {
        float ref = 0;
        for (int k = 0; k < 16; ++k) ref += bf(a_val(mm, 2 * offs[o] + k)) * b_val(n, k);
        if (h_mma[(o * 128 + mm) * 32 + n] != ref) ++bad;
      }
    printf("TS MMA A column offset %3d (elements %3d..): %s (%d/4096 wrong)\n", offs[o], 2 * offs[o],
           bad ? "MISMATCH" : "exact", bad);
  }
  if (mode == 7) {
    int bad = 0;
    auto bits = [](float f) {
      uint32_t u;
      memcpy(&u, &f, 4);
      return u >> 16;
    };
    for (int mm = 0; mm < 128; ++mm)
      for (int j = 0; j < 32; ++j) {
        const uint32_t ex = bits(a_val(mm, 2 * j)) | (bits(a_val(mm, 2 * j + 1)) << 16);
        if (h_cp[mm * 32 + j] != ex) {
          if (bad < 4) printf("  cp lane %d col %d: got %08x want %08x\n", mm, j, h_cp[mm * 32 + j], ex);
          ++bad;
        }
      }
    printf("tcgen05.cp 128x256b from a no-swizzle K-major atom: %s (%d/4096 wrong)\n", bad ? "MISMATCH" : "exact", bad);
    bad = 0;
    for (int mm = 0; mm < 128; ++mm)
      for (int n = 0; n < 32; ++n) {
        float ref = 0;
        for (int k = 0; k < 16; ++k) ref += a_val(mm, k) * b_val(n, k);
        if (h_cpmma[mm * 32 + n] != ref) ++bad;
      }
    printf("MMA on the cp'd A: %s (%d wrong)\n", bad ? "MISMATCH" : "exact", bad);
    return 0;
  }
  if (mode == 8) {
    printf("tcgen05.cp 128x256b (no swizzle): %.1f cyc each (4 KB)\n", cyc[2] / 1024.0);
    return 0;
  }
  if (mode != 1) goto timing;
  {
  int bad = 0;
  for (int mm = 0; mm < 128; ++mm)
    for (int j = 0; j < 32; ++j) {
      // expected: A row mm elements 2j, 2j+1 (bf16 bits)
      auto bits = [](float f) {
        uint32_t u;
        memcpy(&u, &f, 4);
        return u >> 16;
      };
      const uint32_t ex = bits(a_val(mm, 2 * j)) | (bits(a_val(mm, 2 * j + 1)) << 16);
      if (h_cp[mm * 32 + j] != ex) {
        if (bad < 4) printf("  cp lane %d col %d: got %08x want %08x\n", mm, j, h_cp[mm * 32 + j], ex);
        ++bad;
      }
    }
  printf("tcgen05.cp 128x256b from SW128 atom (desc + 32k B): %s (%d/4096 wrong)\n", bad ? "MISMATCH" : "exact", bad);
  bad = 0;
  for (int mm = 0; mm < 128; ++mm)
    for (int n = 0; n < 32; ++n) {
      float ref = 0;
      for (int k = 0; k < 16; ++k) ref += a_val(mm, (the_off == 1 ? 0 : 4) + k) * b_val(n, k);
      if (h_cpmma[mm * 32 + n] != ref) ++bad;
    }
  printf("MMA on cp'd A at column offset 2: %s (%d wrong)\n", bad ? "MISMATCH" : "exact", bad);
  }
timing:
  if (mode == 5 || mode == 6) printf("sweep-like TS rows N=%d (%s): %.1f cyc/MMA\n", the_off, mode == 5 ? "aligned" : "col+8", cyc[0] / (64.0 * 36));
  if (mode == 2 || mode == 3) printf("TS MMA N=96 (%s): %.1f cyc/MMA\n", mode == 2 ? "aligned" : "col+2", cyc[mode - 2] / 2048.0);
  if (mode == 4)
  printf("tcgen05.cp 128x256b: %.1f cyc each (4 KB)\n", cyc[2] / 1024.0);
  return 0;
}
