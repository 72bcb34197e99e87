// window_gemm.cu -- MEC's window GEMMs on tcgen05 / TMEM / TMA (sm_100a).
//
// Paper: every output row h is one GEMM of an overlapping window of L times K
// (Sec. 3.2; Alg.2 l.10-12 and l.23-25):
//
//   Solution A (batch-folded, l.10-12):
//     O[h, 0:i_n o_w k_c] = L[0:i_n o_w, s_h k_w i_c h : + k_h k_w i_c] x K
//   Solution B (per-image, l.23-25):
//     O[n][h, 0:o_w k_c]  = L[n][0:o_w, s_h k_w i_c h : + k_h k_w i_c] x K
//
// The window is a sub-matrix "specified by providing a pointer to the initial
// element and ld".  Here it is a TMA box: a 3-D tensor map over L
// {columns = i_h k_w i_c, rows, groups} with row stride = L's pitch, loaded
// at coordinates (h s_h k_w i_c + k-tile offset, row0, group).  So no
// im2col-sized buffer exists anywhere: the windows are read in place from L.
// Solution A tiles rows over the folded (n, w) index (groups = 1,
// rows = i_n o_w); Solution B over one image's w (groups = i_n, rows = o_w),
// with TMA zero-filling rows past o_w.  Both share this one mainloop, so for
// the same (row, h) they perform bit-identical arithmetic.
//
// Kernel structure (persistent, one CTA per SM, 6 warps):
//   warp 0     TMA producer: A window tile (128 rows x 128 B) + B tile
//              (bn rows of Kt x 128 B) per K-tile into a `stages`-deep ring,
//              128-byte swizzled, mbarrier complete_tx.
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//              (M = 128, N = bn, K = 16 bf16 / 8 tf32 per instruction),
//              fp32 accumulators in TMEM, double-buffered (2 x bn columns)
//              so the epilogue of tile i overlaps the MMAs of tile i+1.
//   warps 2-5  epilogue: tcgen05.ld (32 lanes x 16 columns), fp32 -> bf16
//              (RN-even) or fp32, 128-bit stores to O.  Row (n, w) and output
//              row h give the n-h-w-c address directly -- for Solution A
//              this applies Alg.2 l.17-19's permutation O[n,h] = O_hnwc[h,n]
//              at store time (MEC_SOLA_FIX_EPILOGUE); with out_hnwc the
//              paper's h-n-w-c intermediate is written instead.
// Tile order: N-tile fastest, then h, then the row tile, then the group: the
// CTAs in flight at any time work on neighbouring windows of the same L rows,
// which overlap k_h/s_h-fold, so the re-reads hit L2.
//
// TMA alignment: a box must start 16-byte aligned in dim 0, but window h
// starts at column h*shift (shift = s_h k_w i_c, e.g. 132 bf16 = 264 B for
// AlexNet conv1).  The box starts at x = h*shift - delta instead, delta =
// (h*shift) mod (16/elt), and the MMA uses a copy of K_mat shifted down by
// delta rows (Kt variant delta/delta_step; built by the lowering launch).
// K-tail: the reduction is padded to a multiple of the K-tile (64 bf16 / 32
// fp32).  Columns of the box outside [delta, delta + kdim) (neighbouring,
// finite lowered data, or TMA zero fill past the row end) meet zero rows of
// Kt, so they contribute exactly 0 (inputs must be finite).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "mec_internal.h"
#include "ptx.cuh"
#include "tma_host.h"

namespace mec {
namespace {

constexpr int kThreads = 192;
constexpr int kATileBytes = kBM * kTileKBytes;  // 16 KB

struct GemmParams {
  void* O;
  int64_t o_h, o_w, i_n, k_c;
  int64_t rows, groups, n_mt;
  int64_t shift;
  int vec, delta_step;
  int64_t kc_pad;
  int bk;
  int nk;           // K-tiles per window
  int bn, n_tiles_n;
  int64_t num_tiles;
  int stages;
  uint32_t tmem_cols;
  uint32_t idesc;
  bool out_hnwc;
  bool vec_ok;
};

struct TileCoord {
  int64_t nt, h, mt, g;
};

__device__ __forceinline__ TileCoord decode_tile(const GemmParams& p, int64_t t) {
  TileCoord c;
  c.nt = t % p.n_tiles_n;
  t /= p.n_tiles_n;
  c.h = t % p.o_h;
  t /= p.o_h;
  c.mt = t % p.n_mt;
  c.g = t / p.n_mt;
  return c;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <bool kTF32>
__global__ void __launch_bounds__(kThreads, 1)
    window_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + kSmemAlign - 1) & ~uintptr_t(kSmemAlign - 1));
  const int S = p.stages;
  const uint32_t b_tile_bytes = static_cast<uint32_t>(p.bn) * kTileKBytes;
  unsigned char* smemA = smem;
  unsigned char* smemB = smem + static_cast<size_t>(S) * kATileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smemB + static_cast<size_t>(S) * b_tile_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_dyn(tmem_slot, p.tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t hintA = ptx::policy_evict_normal();
      const uint64_t hintB = ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const TileCoord c = decode_tile(p, t);
        // window start h*shift, rounded down to a 16-byte boundary (TMA rule);
        // the delta-shifted weight copy absorbs the difference
        const int64_t xw = c.h * p.shift;
        const int64_t delta = xw % p.vec;
        const int32_t x0 = static_cast<int32_t>(xw - delta);
        const int32_t y0 = static_cast<int32_t>(c.mt * kBM);
        const int32_t z0 = static_cast<int32_t>(c.g);
        const int32_t n0 = static_cast<int32_t>((delta / p.delta_step) * p.kc_pad + c.nt * p.bn);
        for (int kt = 0; kt < p.nk; ++kt) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], kATileBytes + b_tile_bytes);
          ptx::tma_load_3d(smemA + static_cast<size_t>(stage) * kATileBytes, &tmA, &full[stage],
                           x0 + kt * p.bk, y0, z0, hintA);
          ptx::tma_load_2d(smemB + static_cast<size_t>(stage) * b_tile_bytes, &tmB, &full[stage],
                           kt * p.bk, n0, hintB);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t a_base = ptx::smem_u32(smemA);
    const uint32_t b_base = ptx::smem_u32(smemB);
    for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * p.bn);
      for (int kt = 0; kt < p.nk; ++kt) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t a_addr = a_base + stage * kATileBytes;
          const uint32_t b_addr = b_base + stage * b_tile_bytes;
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 x 32 B = one 128-byte K-tile row
            ptx::mma_ss<kTF32>(d_tmem, ptx::smem_desc_sw128(a_addr + 32 * k),
                               ptx::smem_desc_sw128(b_addr + 32 * k), p.idesc,
                               (kt | k) != 0 ? 1u : 0u);
          }
          ptx::mma_commit(&empty[stage]);
          if (kt == p.nk - 1) ptx::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int quarter = warp & 3;  // TMEM lanes [32 quarter, 32 quarter + 32)
    const int row_in_tile = quarter * 32 + lane;
    constexpr int kOutElt = kTF32 ? 4 : 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      const TileCoord c = decode_tile(p, t);
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int64_t r = c.mt * kBM + row_in_tile;
      const bool valid = r < p.rows;
      const int64_t gr = c.g * p.rows + r;  // flattened (n, w) row of L
      int64_t out_row;
      if (p.out_hnwc) {
        out_row = c.h * (p.i_n * p.o_w) + gr;  // O_hnwc[h, n o_w + w]
      } else {
        const int64_t n = gr / p.o_w, w = gr - n * p.o_w;
        out_row = (n * p.o_h + c.h) * p.o_w + w;  // O[n, h, w]
      }
      unsigned char* orow =
          static_cast<unsigned char*>(p.O) + (out_row * p.k_c + c.nt * p.bn) * kOutElt;
      const int64_t cols_left = p.k_c - c.nt * p.bn;  // valid columns in this N tile
      const uint32_t taddr =
          tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * p.bn);
      for (int c0 = 0; c0 < p.bn; c0 += 16) {
        uint32_t v[16];
        ptx::tmem_ld_32x32b_x16(taddr + c0, v);
        ptx::tmem_ld_wait();
        if (!valid || c0 >= cols_left) continue;
        if constexpr (kTF32) {
          if (p.vec_ok) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (c0 + 4 * j + 4 <= cols_left)
                *reinterpret_cast<uint4*>(orow + (c0 + 4 * j) * 4) =
                    make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
            for (int j = 0; j < 16 && c0 + j < cols_left; ++j)
              reinterpret_cast<uint32_t*>(orow)[c0 + j] = v[j];
          }
        } else {
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            pk[j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
          if (p.vec_ok) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              if (c0 + 8 * j + 8 <= cols_left)
                *reinterpret_cast<uint4*>(orow + (c0 + 8 * j) * 2) =
                    make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          } else {
            for (int j = 0; j < 16 && c0 + j < cols_left; ++j)
              reinterpret_cast<uint16_t*>(orow)[c0 + j] =
                  static_cast<uint16_t>(pk[j >> 1] >> ((j & 1) * 16));
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

}  // namespace

cudaError_t launch_window_gemm(const Plan& pl, const GemmArgs& a, cudaStream_t st,
                               int* launches) {
  const bool tf32 = pl.dt == MEC_DTYPE_TF32;
  CUtensorMap tmA, tmB;
  // A: the lowered tensor L viewed as {columns, rows, groups} (Alg.2 l.9 / l.21).
  {
    const uint64_t dims[3] = {static_cast<uint64_t>(pl.l_cols), static_cast<uint64_t>(a.rows),
                              static_cast<uint64_t>(a.groups)};
    const uint64_t strides[2] = {static_cast<uint64_t>(pl.pitch) * pl.elt,
                                 static_cast<uint64_t>(pl.pitch) * pl.elt * a.rows};
    const uint32_t box[3] = {static_cast<uint32_t>(pl.bk), kBM, 1};
    cudaError_t e = encode_tiled(&tmA, tf32, 3, a.L, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  // B: the prepared weight operand Kt, n_var x kc_pad rows of kdim_pad, K-major.
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(pl.kdim_pad),
                              static_cast<uint64_t>(pl.n_var * pl.kc_pad)};
    const uint64_t strides[1] = {static_cast<uint64_t>(pl.kdim_pad) * pl.elt};
    const uint32_t box[2] = {static_cast<uint32_t>(pl.bk), static_cast<uint32_t>(pl.bn)};
    cudaError_t e = encode_tiled(&tmB, tf32, 2, a.Kt, dims, strides, box);
    if (e != cudaSuccess) return e;
  }

  GemmParams p{};
  p.O = a.O;
  p.o_h = pl.o_h;
  p.o_w = pl.o_w;
  p.i_n = pl.s.i_n;
  p.k_c = pl.s.k_c;
  p.rows = a.rows;
  p.groups = a.groups;
  p.n_mt = (a.rows + kBM - 1) / kBM;
  p.shift = pl.shift;
  p.vec = pl.vec;
  p.delta_step = pl.delta_step;
  p.kc_pad = pl.kc_pad;
  p.bk = pl.bk;
  p.nk = static_cast<int>(pl.kdim_pad / pl.bk);
  p.bn = pl.bn;
  p.n_tiles_n = pl.n_tiles_n;
  p.num_tiles = a.groups * p.n_mt * pl.o_h * pl.n_tiles_n;
  p.out_hnwc = a.out_hnwc;
  p.vec_ok = ((pl.s.k_c * pl.elt) % 16 == 0) && (reinterpret_cast<uintptr_t>(a.O) % 16 == 0);
  p.idesc = ptx::instr_desc(tf32, kBM, pl.bn);
  uint32_t cols = 32;
  while (cols < 2u * pl.bn) cols <<= 1;
  p.tmem_cols = cols;

  const size_t stage_bytes = kATileBytes + static_cast<size_t>(pl.bn) * kTileKBytes;
  const size_t budget = 220 * 1024;
  int stages = static_cast<int>(std::min<size_t>(8, budget / stage_bytes));
  stages = std::max(2, std::min<int>(stages, std::max(2, p.nk * 2)));
  p.stages = stages;
  const size_t smem = kSmemAlign + stages * stage_bytes + (2 * stages + 4) * 8 + 16;

  const int64_t grid = std::min<int64_t>(p.num_tiles, num_sms());
  if (grid <= 0) return cudaSuccess;
  auto kern = tf32 ? window_gemm_kernel<true> : window_gemm_kernel<false>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(tmA, tmB, p);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace mec
