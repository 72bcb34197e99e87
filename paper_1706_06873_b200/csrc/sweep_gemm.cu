// sweep_gemm.cu -- MEC's window GEMMs as a sweep along h, A staged in TMEM
// (sm_100a).
//
// Paper: output row h is O[:, h] = L[:, h s_h k_w i_c : + k_h k_w i_c] x K,
// one GEMM per row over an overlapping window of L (Sec. 3.2, P:100-102;
// Alg.2 l.10-12 Solution A, l.23-25 Solution B).  Consecutive windows overlap
// by k_h k_w i_c - s_h k_w i_c columns: the paper's BLAS calls re-read that
// overlap once per row (k_h / s_h times in all).  On B200 the re-reads come
// from L2, whose bandwidth to the SMs is about the HBM bandwidth, so the
// one-window-per-tile schedule (window_gemm.cu) is bounded by ~(k_h/s_h) #L
// of L2 traffic, not by #L.
//
// This kernel streams each 128-row tile of L ONCE along its columns and
// lets every output row h take its window out of the stream:
//   * a work item is (row tile, a chunk of H consecutive output rows); its
//     stream is the column range [x0, (h_end - 1) shift + kdim) of the tile's
//     L rows, read as 128-byte K-atoms by TMA into a shared-memory ring;
//   * 4 copier warps move each atom from shared memory into a TMEM ring
//     (tcgen05.st, row m -> TMEM lane m), so the MMAs take A from TMEM (the
//     "TS" form).  A TMEM operand can start at any 16-byte column step, so
//     row h's window is addressed at its exact offset o = h shift - x0 up to
//     d = o mod (16 B / elt) elements; d is absorbed by the weight copy
//     shifted down by d rows (Kt variant d / delta_step, mec_internal.h).
//     All the variants needed (at most 16 B / gcd(shift elt, 16 B)) stay
//     resident in shared memory;
//   * one thread issues, when atom i has landed, every 32-byte K step of every
//     open row whose last element falls in atom i (a step that straddles two
//     atoms reads a TMEM guard copy of the next atom's first 16 bytes when the
//     ring wraps); rows use a ring of TMEM accumulators, opened at their first
//     step and committed to the epilogue at their last;
//   * 8 epilogue warps (two groups, alternate rows) drain the accumulators
//     row by row: tcgen05.ld -> bf16/fp32 -> swizzled smem -> TMA store of
//     O[n, h, w, :] (n-h-w-c; Solution A's permutation, Alg.2 l.17-19, applied
//     at store time) or of O_hnwc[h, n, w, :] (the paper's intermediate).
// L2 -> SM traffic per item: (H - 1) shift + kdim columns instead of
// H kdim.  Per row the arithmetic is the same K steps, in the same order, for
// Solution A and B (so A == B bitwise, reading Q10).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "mec_internal.h"
#include "ptx.cuh"
#include "tma_host.h"

#ifdef MEC_TRACE
// Debug-only per-atom timestamps (tools/trace_sweep.py, -DMEC_TRACE build):
// [cta < 160][atom seq < 256][event < 8]
__device__ unsigned long long* g_sweep_trace = nullptr;
extern "C" int mec_sweep_trace_enable(void** dev_buf_out, size_t* bytes_out) {
  const size_t bytes = static_cast<size_t>(160) * 512 * 8 * 8;
  void* buf = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
  cudaMemset(buf, 0, bytes);
  if (cudaMemcpyToSymbol(g_sweep_trace, &buf, sizeof(buf)) != cudaSuccess) return 2;
  *dev_buf_out = buf;
  *bytes_out = bytes;
  return 0;
}
#define SW_TRACE(seq, ev)                                                                      \
  do {                                                                                         \
    if (sw_tr != nullptr && blockIdx.x < 160 && (seq) < 512) {                                 \
      unsigned long long t_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      sw_tr[(static_cast<size_t>(blockIdx.x) * 512 + (seq)) * 8 + (ev)] = t_;                  \
    }                                                                                          \
  } while (0)
#else
#define SW_TRACE(seq, ev) \
  do {                    \
  } while (0)
#endif

namespace mec {
namespace {

// copier warps in groups of 4 (one per 32-row quarter; groups take alternate
// atoms) and epilogue warps in groups of 4 (groups take alternate rows).
// Default 1 copier group + 2 epilogue groups; 2 + 1 (-DMEC_SW_COPY_GROUPS=2
// -DMEC_SW_EPI_GROUPS=1) measured slower: C2 GEMM 319 vs 315 us, cv3 b128
// 125 vs 89 us, cv7 391 vs 241 us (one epilogue group cannot keep up with
// short windows).
#ifndef MEC_SW_COPY_GROUPS
#define MEC_SW_COPY_GROUPS 1
#endif
#ifndef MEC_SW_EPI_GROUPS
#define MEC_SW_EPI_GROUPS 2
#endif
constexpr int kSwCopyGroups = MEC_SW_COPY_GROUPS;
constexpr int kSwEpiGroups = MEC_SW_EPI_GROUPS;
constexpr int kSwCopyWarps = 4 * kSwCopyGroups;
constexpr int kSwEpiWarps = 4 * kSwEpiGroups;
constexpr int kSwFirstCopyWarp = 2;
constexpr int kSwFirstEpiWarp = kSwFirstCopyWarp + kSwCopyWarps;
// MMA issuer warps (rows dealt round-robin, p.n_iss = 1 or 2; the second is
// warp kSwMma2Warp): a second issuer overlaps one row's per-row control code
// with the other's MMAs (single-warp issue is latency-bound).
constexpr int kSwMaxIssuers = 2;
constexpr int kSwMma2Warp = kSwFirstEpiWarp + kSwEpiWarps;
constexpr int kSwThreads = 32 * (kSwMma2Warp + 1);  // 480 (2 copier groups + 1 epilogue group, or 1 + 2)
constexpr int kSwAtomBytes = kBM * kTileKBytes;                   // 16 KB: 128 rows x 128 B
constexpr int kSwMaxRing = 16;
constexpr int kSwMaxAcc = 8;
constexpr int kSwGuardCols = 32;  // TMEM guard after the A ring: a copy of slot 0's atom

struct SweepParams {
  void* O;
  int64_t o_h, o_w, i_n, k_c;
  // row tiling, as in window_gemm.cu: flat (Solution A, o_w < 32: 128 folded
  // rows n o_w + w per tile), packed (ipt images per tile in `slot`-row
  // slots) or one image per tile (ipt = 1)
  bool flat;
  int ipt, slot;
  int64_t rows, groups, n_mt;
  int shift;       // s_h k_w i_c (elements)
  int kdim;        // k_h k_w i_c
  int bk;          // K-atom (elements per 128 B)
  int bk_log2;
  int kchunk_log2; // elements per 32-byte MMA K step: 16 bf16 / 8 tf32
  int mvec;        // elements per 16 bytes (TMEM A operand column step)
  int avec;        // TMA box-start alignment of x0 (elements)
  int ds_log2;     // log2(delta_step): variant v = d / delta_step
  int nb_atoms;    // B atoms per weight variant (kdim_pad / bk)
  int n_vres;      // resident weight variants
  int64_t kc_pad;
  int bn;
  int H;           // output rows of the largest work item (chunks differ by <= 1 row)
  int64_t n_hc, n_items;
  // balanced split (bal_G > 0): CTA c owns rows [c R / G, (c + 1) R / G) of
  // the flattened (tile, h) sequence (R = n_tiles o_h), cut at tile
  // boundaries into at most bal_J items; item t = c + j G is piece j of CTA c
  int64_t bal_R;
  int bal_G, bal_J;
  int stages;      // shared-memory A stages (one atom each)
  int ns;          // TMEM A ring slots (32 columns each)
  int n_acc;       // TMEM accumulators (bn columns each)
  uint32_t a_col0, guard_col;
  uint32_t idesc;
  int col_shift;   // TMEM column of element e within an atom: (e mod bk) >> col_shift... (bf16: 1, tf32: 0)
  bool out_hnwc;
  bool tma_store;
  int pw, n_pass;
  uint32_t stage_out_bytes;
  uint32_t backoff_ns;  // copier / epilogue waits: nanosleep between probes (0: spin)
  int n_iss;  // MMA issuer warps (1 or 2)
  // A into the TMEM ring by tcgen05.cp issued from the MMA thread (DESIGN.md
  // 6.2b): no copier warps; the copies and the MMAs execute in issue order
  bool cp;
  // CTA-pair mode (kPair kernels): CTA tiles are dealt in
  // pairs (CTA rank r takes tile 2 pt + r); n_tiles = n_mt groups
  int64_t n_tiles;
  // fused (MEC_PATH_FUSED, i_c elt a multiple of 128 B): stream atoms are TMA
  // boxes of I -- column c = hh kwc + b i_c + ci of L row (n, w) is pixel
  // s_w w + b of input row hh, channels ci (Alg.2 l.4-6), so L is never written
  bool fused;
  int kwc, i_c, s_w, pad_h, pad_w;
  int dbg;  // (experiments, MEC_SWEEP_DBG) 1: no O stores, 2: no MMAs, 4: no TMEM stores of A
  // tiles in reverse order: the first wave streams the images the lowering
  // wrote last, whose L lines are still in L2
  bool reverse;
};

struct SwItem {
  int64_t h0, mt, g;
  bool valid;  // pair mode: an odd tile count leaves the last pair's second CTA without rows
  int nrows;
  int n_a;     // atoms streamed
  int x0;      // stream start column (multiple of avec)
  int off0;    // h0 shift - x0 (< avec)
};

__device__ __forceinline__ SwItem sw_decode(const SweepParams& p, int64_t t, bool pair = false,
                                           uint32_t rank = 0) {
  SwItem it;
  if (!pair && p.bal_G > 0) {
    const int64_t c0 = t % p.bal_G, j = t / p.bal_G;
    const int64_t c = p.reverse ? p.bal_G - 1 - c0 : c0;
    const int64_t s = c * p.bal_R / p.bal_G, e = (c + 1) * p.bal_R / p.bal_G;
    const int64_t tile0 = s / p.o_h;
    const int64_t start = j == 0 ? s : (tile0 + j) * p.o_h;
    const int64_t end = min(e, (tile0 + j + 1) * p.o_h);
    it.valid = true;
    const int64_t tl = start < end ? start / p.o_h : tile0;
    it.mt = tl % p.n_mt;
    it.g = tl / p.n_mt;
    it.h0 = start < end ? start - tl * p.o_h : 0;
    it.nrows = start < end ? static_cast<int>(end - start) : 0;
  } else {
  // 32-bit index math (items, tiles and rows all fit; 64-bit divisions cost
  // every role ~1 us per item before its first atom, trace build on C1)
  uint32_t tt = static_cast<uint32_t>(t);
  const uint32_t n_hc = static_cast<uint32_t>(p.n_hc), o_h = static_cast<uint32_t>(p.o_h);
  const uint32_t hc = tt % n_hc;
  tt /= n_hc;
  if (pair) tt = 2 * tt + rank;  // pair tile -> this CTA's tile
  else if (p.reverse) tt = static_cast<uint32_t>(p.n_tiles) - 1 - tt;
  it.valid = tt < static_cast<uint32_t>(p.n_tiles);
  if (!it.valid) tt = static_cast<uint32_t>(p.n_tiles) - 1;  // (a real tile's coordinates; nothing is stored)
  const uint32_t n_mt = static_cast<uint32_t>(p.n_mt);
  it.mt = tt % n_mt;
  it.g = tt / n_mt;
  // chunk hc: rows [hc o_h / n_hc, (hc + 1) o_h / n_hc) (sizes differ by <= 1)
  const uint32_t h0 = hc * o_h / n_hc;
  it.h0 = h0;
  it.nrows = static_cast<int>((hc + 1) * o_h / n_hc - h0);
  }
  const uint32_t xs = static_cast<uint32_t>(it.h0) * static_cast<uint32_t>(p.shift);  // < 2^30 (sweep_config)
  it.x0 = static_cast<int>(xs - xs % static_cast<uint32_t>(p.avec));
  it.off0 = static_cast<int>(xs - static_cast<uint32_t>(it.x0));
  if (it.nrows == 0) {  // (an empty piece of a balanced split: no atoms, no rows)
    it.n_a = 0;
    return it;
  }
  // the last row's last K step bounds the stream
  const int o_last = it.off0 + (it.nrows - 1) * p.shift;
  const int d_last = o_last & (p.mvec - 1);
  const int kc = 1 << p.kchunk_log2;
  // (a row's K steps are rounded up to whole 4-step groups: the extra steps
  // meet zero weight rows, see the MMA issuer)
  const int nk_last = (((p.kdim + d_last + kc - 1) >> p.kchunk_log2) + 3) & ~3;
  it.n_a = (o_last - d_last + nk_last * kc + p.bk - 1) / p.bk;
  return it;
}

__device__ __forceinline__ uint32_t sw_pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Epilogue of one output row h of tile (mt, g): this warp's 32 TMEM lanes
// (quarter) of accumulator columns taddr .. taddr + bn.  Same stores as the
// one-window-per-tile kernel.
template <bool kTF32>
// The accumulator is released (tempty arrive) as soon as the last pass's
// tcgen05.ld has completed, before the conversion and the stores, so the
// next row that uses it can start accumulating while this one is stored.
__device__ __forceinline__ void sw_store_row(const SweepParams& p, const CUtensorMap* tmO, int64_t h, int64_t mt,
                                             int64_t g, int quarter, int lane, uint32_t taddr, uint32_t stg,
                                             unsigned char* stg_gen, uint64_t* tempty_bar, bool valid = true,
                                             uint32_t tempty_cluster = 0) {
  constexpr int kOutElt = kTF32 ? 4 : 2;
  const int row_bytes = p.pw * kOutElt;
  const int swz_shift = row_bytes == 128 ? 0 : (row_bytes == 64 ? 1 : 2);
  const int swz_mask = row_bytes == 128 ? 7 : (row_bytes == 64 ? 3 : 1);
  const uint32_t my_x = static_cast<uint32_t>((lane >> swz_shift) & swz_mask);
  int64_t gr0, nvalid, n_img = 0, w0 = 0;
  if (p.flat) {
    const int64_t r0 = mt * kBM + quarter * 32;
    nvalid = min(static_cast<int64_t>(32), p.rows - r0);
    gr0 = r0;
  } else {
    const int j = (quarter * 32) / p.slot;
    n_img = g * p.ipt + j;
    w0 = mt * kBM + quarter * 32 - j * p.slot;
    nvalid = (j < p.ipt && n_img < p.i_n) ? min(static_cast<int64_t>(32), p.o_w - w0) : 0;
    gr0 = n_img * p.o_w + w0;
  }
  if (!valid) nvalid = 0;
  unsigned char* orow_own;
  {
    const int64_t gr = gr0 + lane;
    int64_t out_row;
    if (p.out_hnwc) {
      out_row = h * (p.i_n * p.o_w) + gr;
    } else {
      // (32-bit division: i_n o_w < 2^31, launch_sweep_gemm)
      const uint32_t n = static_cast<uint32_t>(gr) / static_cast<uint32_t>(p.o_w);
      const int64_t w = gr - static_cast<int64_t>(n) * p.o_w;
      out_row = (static_cast<int64_t>(n) * p.o_h + h) * p.o_w + w;
    }
    orow_own = static_cast<unsigned char*>(p.O) + out_row * p.k_c * kOutElt;
  }
  for (int pass = 0; pass < p.n_pass; ++pass) {
    const int c0 = pass * p.pw;
    uint32_t v16[4][16];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j * 16 < p.pw) ptx::tmem_ld_32x32b_x16(taddr + c0 + 16 * j, v16[j]);
    ptx::tmem_ld_wait();
    if (pass == p.n_pass - 1) {
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (tempty_cluster != 0) ptx::mbar_arrive_cluster(tempty_cluster);  // the pair leader's barrier
        else ptx::mbar_arrive(tempty_bar);
      }
    }
    if (nvalid <= 0 || c0 >= p.k_c || (p.dbg & 1)) continue;  // warp-uniform
    if (p.tma_store) {
      const uint32_t my_row = stg + static_cast<uint32_t>(lane * row_bytes);
      if (lane == 0) ptx::bulk_wait_group_read<0>();  // the previous store finished reading the box
      __syncwarp();
      const int nchunk = row_bytes / 16;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        if (ch >= nchunk) break;
        uint32_t q0, q1, q2, q3;
        if constexpr (kTF32) {
          const int j = ch >> 2, e = (ch & 3) * 4;
          q0 = v16[j][e];
          q1 = v16[j][e + 1];
          q2 = v16[j][e + 2];
          q3 = v16[j][e + 3];
        } else {
          const int j = ch >> 1, e = (ch & 1) * 8;
          q0 = sw_pack_bf16x2(__uint_as_float(v16[j][e]), __uint_as_float(v16[j][e + 1]));
          q1 = sw_pack_bf16x2(__uint_as_float(v16[j][e + 2]), __uint_as_float(v16[j][e + 3]));
          q2 = sw_pack_bf16x2(__uint_as_float(v16[j][e + 4]), __uint_as_float(v16[j][e + 5]));
          q3 = sw_pack_bf16x2(__uint_as_float(v16[j][e + 6]), __uint_as_float(v16[j][e + 7]));
        }
        ptx::st_shared_v4(my_row + ((static_cast<uint32_t>(ch) ^ my_x) << 4), q0, q1, q2, q3);
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      const int32_t col = c0;
      if (!p.flat) {
        if (lane == 0) {
          if (p.out_hnwc)  // O_hnwc as {k_c, o_w, i_n, o_h}
            ptx::tma_store_4d(tmO, stg_gen, col, static_cast<int32_t>(w0), static_cast<int32_t>(n_img),
                              static_cast<int32_t>(h));
          else  // O as {k_c, o_w, o_h, i_n}
            ptx::tma_store_4d(tmO, stg_gen, col, static_cast<int32_t>(w0), static_cast<int32_t>(h),
                              static_cast<int32_t>(n_img));
          ptx::bulk_commit_group();
        }
      } else if (p.out_hnwc) {
        if (lane == 0) {
          ptx::tma_store_3d(tmO, stg_gen, col, static_cast<int32_t>(gr0), static_cast<int32_t>(h));
          ptx::bulk_commit_group();
        }
      } else {
        // rows of the first image: one TMA store; rows of a later image in the
        // 32-row block (TMA stores reject negative coordinates) by the warp
        const int64_t n_first = gr0 / p.o_w;
        const int k_first = static_cast<int>(min(nvalid, (n_first + 1) * p.o_w - gr0));
        if (lane == 0) {
          ptx::tma_store_4d(tmO, stg_gen, col, static_cast<int32_t>(gr0 - n_first * p.o_w),
                            static_cast<int32_t>(h), static_cast<int32_t>(n_first));
          ptx::bulk_commit_group();
        }
        if (k_first < nvalid) {
          const int lg = nchunk == 8 ? 3 : (nchunk == 4 ? 2 : 1);
          const int nrest = static_cast<int>(nvalid) - k_first;
          const int total = nrest * nchunk;
          for (int ci0 = 0; ci0 < total; ci0 += 32) {
            const int ci = min(ci0 + lane, total - 1);
            const int row = k_first + (ci >> lg), ch = ci & (nchunk - 1);
            const unsigned long long base =
                __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(orow_own), row);
            const uint32_t x = static_cast<uint32_t>((row >> swz_shift) & swz_mask);
            const uint4 val =
                ptx::ld_shared_v4(stg + static_cast<uint32_t>(row * row_bytes) + ((static_cast<uint32_t>(ch) ^ x) << 4));
            if (ci0 + lane < total)
              *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(base) + c0 * kOutElt + ch * 16) = val;
          }
        }
      }
    } else if (lane < nvalid) {
      // k_c elt not a multiple of 16 (or of the pass width): element stores
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int col = c0 + j * 16 + e;
          if (j * 16 + e < p.pw && col < p.k_c) {
            if constexpr (kTF32) {
              reinterpret_cast<uint32_t*>(orow_own)[col] = v16[j][e];
            } else {
              const uint32_t pkd = sw_pack_bf16x2(__uint_as_float(v16[j][e]), 0.0f);
              reinterpret_cast<uint16_t*>(orow_own)[col] = static_cast<uint16_t>(pkd & 0xFFFFu);
            }
          }
        }
      }
    }
  }
}

template <bool kTF32, bool kPair>
__global__ void __launch_bounds__(kSwThreads, 1)
    sweep_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, const SweepParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + kSmemAlign - 1) & ~uintptr_t(kSmemAlign - 1));
  const int S = p.stages;
  // pair mode: each CTA holds bn / 2 rows of every weight atom (the pair's MMA
  // reads N/2 columns of B from each CTA)
  const uint32_t b_tile_bytes = static_cast<uint32_t>(kPair ? p.bn / 2 : p.bn) * kTileKBytes;
  const int n_btiles = p.n_vres * p.nb_atoms;
  unsigned char* smemA = smem;
  unsigned char* smemB = smem + static_cast<size_t>(S) * kSwAtomBytes;
  unsigned char* smemE = smemB + static_cast<size_t>(n_btiles) * b_tile_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smemE + static_cast<size_t>(kSwEpiWarps) * p.stage_out_bytes);
  uint64_t* full = bars;                    // [S]  TMA -> copiers
  uint64_t* empty = bars + 8;               // [S]  copiers -> TMA
  uint64_t* afull = bars + 16;              // [ns] copiers -> MMA
  // rows completed, per epilogue group (even / odd global row numbers):
  // epilogue -> copiers.  A slot is refilled once the last row that reads its
  // atom has completed; monotonic counters instead of per-slot barriers keep
  // the MMA warp at one tcgen05.commit per row (a commit costs ~500 cycles)
  uint32_t* rows_done = reinterpret_cast<uint32_t*>(bars + 32);
  uint64_t* tfull = bars + 48;              // [n_acc] MMA -> epilogue
  uint64_t* tempty = bars + 56;             // [n_acc] epilogue -> MMA
  uint64_t* bfull = bars + 64;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 65);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? ptx::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int64_t t_begin = kPair ? static_cast<int64_t>(ptx::cluster_id_x()) : static_cast<int64_t>(blockIdx.x);
  const int64_t t_step = kPair ? static_cast<int64_t>(ptx::nclusters_x()) : static_cast<int64_t>(gridDim.x);
#ifdef MEC_TRACE
  unsigned long long* const sw_tr = g_sweep_trace;
#endif

  if (threadIdx.x == 0) SW_TRACE(511u, 0);
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    ptx::tma_prefetch_desc(&tmO);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], p.cp ? 1 : 4);  // one copier group; cp mode: one tcgen05.commit per atom
    }
    // (pair mode: the leader's ring barriers count both CTAs' copier warps)
    for (int i = 0; i < p.ns; ++i) ptx::mbar_init(&afull[i], 4 * (kPair ? 2 : 1));
    rows_done[0] = 0;
    rows_done[1] = 0;
    for (int i = 0; i < p.n_acc; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kPair ? 8 : 4);  // the 4 warps of an epilogue group (x 2 CTAs)
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (kPair) ptx::tmem_alloc_pair(tmem_slot, 512);
    else ptx::tmem_alloc_dyn(tmem_slot, 512);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kPair) ptx::cluster_sync();  // both CTAs' barriers initialised (remote arrives follow)
  ptx::tc_fence_after();
  // broadcast from lane 0: provably warp-uniform, so the MMA warp keeps its
  // operand addresses in uniform registers (no per-MMA R2UR loops)
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  if (threadIdx.x == 0) SW_TRACE(511u, 1);

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t hintA = ptx::policy_evict_normal();
      const uint64_t hintB = ptx::policy_evict_last();
      ptx::griddep_wait();  // L and Kt come from the preceding (lowering) kernel
      if (t_begin < p.n_items) {
        ptx::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(n_btiles) * b_tile_bytes);
        for (int v = 0; v < p.n_vres; ++v)
          for (int a = 0; a < p.nb_atoms; ++a)
            ptx::tma_load_2d(smemB + static_cast<size_t>(v * p.nb_atoms + a) * b_tile_bytes, &tmB, bfull, a * p.bk,
                             static_cast<int32_t>(v * p.kc_pad + (kPair ? rank * (p.bn / 2) : 0)), hintB);
      }
      SW_TRACE(511u, 2);
      uint32_t pseq = 0;
      int stage = 0;
      uint32_t pphase = 0;
      for (int64_t t = t_begin; t < p.n_items; t += t_step) {
        const SwItem it = sw_decode(p, t, kPair, rank);
        const int32_t y0 = static_cast<int32_t>(it.mt * kBM);
        const int32_t z0 = static_cast<int32_t>(it.g);
        // fused: L column x -> input row hh, kernel column b, channel block cb,
        // advanced by one atom (bk channels; i_c is a multiple of bk) per step
        // -- no divisions on the per-atom path
        int f_hh = 0, f_b = 0, f_cb = 0;
        if (p.fused) {
          f_hh = it.x0 / p.kwc;
          const int rem = it.x0 - f_hh * p.kwc;
          f_b = rem / p.i_c;
          f_cb = rem - f_b * p.i_c;
        }
        for (int i = 0; i < it.n_a; ++i, ++pseq) {
          if (pseq < 100) SW_TRACE(300u + pseq, 0);
          ptx::mbar_wait(&empty[stage], pphase ^ 1u);
          if (pseq < 100) SW_TRACE(300u + pseq, 1);
          ptx::mbar_arrive_expect_tx(&full[stage], kSwAtomBytes);
          unsigned char* dstA = smemA + static_cast<size_t>(stage) * kSwAtomBytes;
          const int32_t x = it.x0 + i * p.bk;
          if (p.fused) {
            // L column x -> input row hh, kernel column b, channel block cb
            const int hh = f_hh, b = f_b, cb = f_cb;
            if ((f_cb += p.bk) == p.i_c) {
              f_cb = 0;
              if (++f_b == p.kwc / p.i_c) {
                f_b = 0;
                ++f_hh;
              }
            }
            const int32_t zy = hh - p.pad_h;  // (padding: TMA zero-fills out-of-bounds pixels and rows)
            // (ipt > 1: one box of ipt images x `slot` pixels -- the box's
            // last extent is ipt; images >= i_n and pixels >= the width: zero fill)
            ptx::tma_load_4d(dstA, &tmA, &full[stage], cb, (p.ipt <= 1 ? y0 * p.s_w : 0) + b - p.pad_w, zy,
                             p.ipt <= 1 ? z0 : z0 * p.ipt, hintA);
          } else if (p.ipt <= 1) {
            ptx::tma_load_3d(dstA, &tmA, &full[stage], x, y0, z0, hintA);
          } else {  // one box of ipt images x `slot` rows (images >= i_n, rows >= o_w: zero fill)
            ptx::tma_load_3d(dstA, &tmA, &full[stage], x, 0, z0 * p.ipt, hintA);
          }
          SW_TRACE(pseq, 0);
          if (pseq < 100) SW_TRACE(300u + pseq, 2);
          if (++stage == S) {
            stage = 0;
            pphase ^= 1u;
          }
        }
      }
    }
  } else if (p.cp && warp == 1 && leader) {
    // ===================== MMA issuer with tcgen05.cp (cp mode) =====================
    // One thread copies each landed atom from its shared-memory stage into the
    // TMEM ring (4 x tcgen05.cp.128x256b of the SW128 atom, + the guard copy
    // of slot 0) and issues the rows.  Copies and MMAs of one thread execute
    // in issue order, so a ring slot is rewritten only after the MMAs issued
    // before (the rows that read its previous atom) have read it: no slot
    // counters.  Atoms are copied just before the first row that needs them.
    const uint64_t b_desc0 = ptx::smem_desc_sw128(ptx::smem_u32(smemB));
    const uint64_t a_sdesc0 = ptx::smem_desc_sw128(ptx::smem_u32(smemA));
    const uint32_t b_tile16 = b_tile_bytes >> 4;
    const uint32_t bvar16 = b_tile16 * static_cast<uint32_t>(p.nb_atoms);
    const int kcl = p.kchunk_log2, cs = p.col_shift, bkl = p.bk_log2;
    const int ns = p.ns, shift = p.shift, mmask = p.mvec - 1;
    const int kdim_r = p.kdim + (1 << kcl) - 1;
    const uint32_t ring0 = tmem_base + p.a_col0, ring_cols = static_cast<uint32_t>(32 * ns);
    const bool no_mma = (p.dbg & 2) != 0;
    if (t_begin < p.n_items) ptx::mbar_wait(bfull, 0);
    int stage = 0, ring = 0;  // next atom's smem stage and TMEM ring slot
    uint32_t sphase = 0;
    uint32_t q = 0;  // global sequence number of the item's row 0
    for (int64_t t = t_begin; t < p.n_items; t += t_step) {
      const SwItem it = sw_decode(p, t, kPair, rank);
      const int slot0 = ring;  // ring slot of the item's atom 0
      int cp_next = 0;         // next atom of the item to copy
      auto copy_atom = [&]() {
        ptx::mbar_wait(&full[stage], sphase);
        ptx::tc_fence_after();
        const uint64_t src = a_sdesc0 + (static_cast<uint32_t>(stage * kSwAtomBytes) >> 4);
        if (!(p.dbg & 4)) {
          ptx::tmem_cp_atom_elect(ring0 + static_cast<uint32_t>(ring * 32), src);
          if (ring == 0) ptx::tmem_cp_atom_elect(tmem_base + p.guard_col, src);  // guard
        }
        ptx::mma_commit_elect(&empty[stage]);  // the stage is free once the copies have read it
        __syncwarp();
        if (++stage == p.stages) {
          stage = 0;
          sphase ^= 1u;
        }
        if (++ring == ns) ring = 0;
        ++cp_next;
      };
      int o = it.off0;
      for (int r = 0; r < it.nrows; ++r, o += shift) {
        const int d = o & mmask;
        const int a = o - d;  // stream element of the row's first step
        const int nk = (kdim_r + d) >> kcl;
        const int n_full = (nk + 3) >> 2;
        const int last = (a + (n_full << (kcl + 2)) - 1) >> bkl;  // last atom the row reads
        while (cp_next <= last) copy_atom();
        const uint32_t g = q + static_cast<uint32_t>(r);
        const int acc = p.n_acc == 2 ? static_cast<int>(g & 1u) : 0;
        const uint32_t acc_use = p.n_acc == 2 ? (g >> 1) : g;
        ptx::mbar_wait(&tempty[acc], (acc_use & 1u) ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * p.bn);
        int s0 = slot0 + (a >> bkl);
        while (s0 >= ns) s0 -= ns;
        const uint32_t col = ring0 + static_cast<uint32_t>(s0 * 32) + (static_cast<uint32_t>(a & ((1 << bkl) - 1)) >> cs);
        const uint64_t bvar = b_desc0 + static_cast<uint32_t>(d >> p.ds_log2) * bvar16;
        if (n_full > 0 && !no_mma)
          // every atom the row needs is copied (issued before these MMAs): no waits in the loop
          ptx::mma_ts_row_elect<kTF32, kPair>(d_tmem, col, ring0 + ring_cols, ring_cols, static_cast<uint32_t>(bvar),
                                              b_tile16, p.idesc, n_full, a, kcl + 2, bkl, ptx::smem_u32(full), 0, 0u,
                                              1 << 30, ns);
        if constexpr (kPair) ptx::mma_commit_pair_elect(&tfull[acc], 0x3);
        else ptx::mma_commit_elect(&tfull[acc]);
        __syncwarp();
      }
      while (cp_next < it.n_a) copy_atom();  // atoms no row reads (the stream's rounding): release them
      ring = slot0 + it.n_a;
      while (ring >= ns) ring -= ns;
      q += static_cast<uint32_t>(it.nrows);
    }
  } else if (p.cp && (warp == 1 || warp == kSwMma2Warp || warp < kSwFirstEpiWarp)) {
    // (cp mode: no copier warps, no second issuer)
  } else if ((warp == 1 || (warp == kSwMma2Warp && p.n_iss > 1)) && leader) {
    // ===================== MMA issuer(s) =====================
    // Issuer mi takes the rows with global sequence number g = mi (mod
    // p.n_iss); row g accumulates into accumulator g mod 2.  A row's K
    // steps (kdim + d elements in 32-byte steps) are issued back to back, 4
    // per election, waiting for each atom as its steps need it; atoms before
    // the row's first are released first (an atom's slot is refilled once
    // every issuer released it).  Single-warp control code is latency-bound
    // (DESIGN.md section 7), so per group of 4 steps the loop does two adds:
    // consecutive groups are 32 TMEM columns apart (the ring wraps; a group
    // across the wrap reads the guard) and one B atom apart.
    const int mi = warp == 1 ? 0 : 1;
    const uint64_t b_desc0 = ptx::smem_desc_sw128(ptx::smem_u32(smemB));
    const uint32_t b_tile16 = b_tile_bytes >> 4;
    const uint32_t bvar16 = b_tile16 * static_cast<uint32_t>(p.nb_atoms);  // descriptor step per weight variant
    const int kcl = p.kchunk_log2, cs = p.col_shift, bkl = p.bk_log2;
    const int ns = p.ns, shift = p.shift, mmask = p.mvec - 1;
    const int kdim_r = p.kdim + (1 << kcl) - 1;
    const uint32_t ring0 = tmem_base + p.a_col0, ring_cols = static_cast<uint32_t>(32 * ns);
    const bool no_mma = (p.dbg & 2) != 0;
    if (t_begin < p.n_items) ptx::mbar_wait(bfull, 0);
    if (lane == 0 && mi == 0) SW_TRACE(511u, 3);
    int wslot = 0;          // ring slot of the next atom to wait for
    uint32_t wphase = 0;
    uint32_t q = 0;         // global sequence number of the item's row 0
    uint32_t aseq = 0;      // atoms waited (traces only)
    (void)aseq;
#ifdef MEC_TRACE
    long long cyc_wait = 0, cyc_issue = 0, cyc_tempty = 0, cyc_row0 = 0;
#endif
    for (int64_t t = t_begin; t < p.n_items; t += t_step) {
      const SwItem it = sw_decode(p, t, kPair, rank);
      const int slot0 = wslot;  // ring slot of the item's atom 0
      int avail = 0;            // atoms of the item landed in TMEM
      int released = 0;         // atoms of the item released by this issuer
      auto wait_atom = [&]() {
#ifdef MEC_TRACE
        const long long cw0 = clock64();
#endif
        ptx::mbar_wait(&afull[wslot], wphase);
#ifdef MEC_TRACE
        cyc_wait += clock64() - cw0;
#endif
        if (lane == 0 && mi == 0 && !(p.dbg & 16)) SW_TRACE(aseq, 4);
        ++aseq;
        if (++wslot == ns) {
          wslot = 0;
          wphase ^= 1u;
        }
        ++avail;
      };
      // advance the ring position over atoms this issuer does not read,
      // without waiting for them (a wait could see their slot refilled twice)
      auto skip_to = [&](int upto) {
        while (avail < upto) {
          if (++wslot == ns) {
            wslot = 0;
            wphase ^= 1u;
          }
          ++avail;
          ++aseq;
        }
      };
      // first row of this issuer: g = q + r = mi (mod n_iss)
      const int n_iss = p.n_iss;
      int r = static_cast<int>((static_cast<uint32_t>(mi + n_iss) - q % n_iss) % n_iss);
      int o = it.off0 + r * shift;
      for (; r < it.nrows; r += n_iss, o += n_iss * shift) {
        const int d = o & mmask;
        const int a = o - d;  // stream element of the row's first step
        const int nk = (kdim_r + d) >> kcl;
        skip_to(a >> bkl);  // atoms before this row's window
        const uint32_t g = q + static_cast<uint32_t>(r);
        // accumulator of row g: g mod n_acc (n_acc = 1 or 2); phase (g / n_acc) mod 2
        const int acc = p.n_acc == 2 ? static_cast<int>(g & 1u) : 0;
        const uint32_t acc_use = p.n_acc == 2 ? (g >> 1) : g;
#ifdef MEC_TRACE
        cyc_wait = 0;
        cyc_issue = 0;
        cyc_row0 = clock64();
#endif
        if constexpr (kPair) ptx::mbar_wait_cluster(&tempty[acc], (acc_use & 1u) ^ 1u);
        else ptx::mbar_wait(&tempty[acc], (acc_use & 1u) ^ 1u);
#ifdef MEC_TRACE
        cyc_tempty = clock64() - cyc_row0;
#endif
        ptx::tc_fence_after();
        if (lane == 0 && mi == 0 && !(p.dbg & 16)) SW_TRACE(static_cast<uint32_t>(r), 6);
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * p.bn);
        // TMEM column of step 0: slot of atom a / bk, then the offset inside it
        int s0 = slot0 + (a >> bkl);
        while (s0 >= ns) s0 -= ns;
        uint32_t col = ring0 + static_cast<uint32_t>(s0 * 32) + (static_cast<uint32_t>(a & ((1 << bkl) - 1)) >> cs);
        const uint64_t bvar = b_desc0 + static_cast<uint32_t>(d >> p.ds_log2) * bvar16;
        // issue the row's full groups in runs: every group whose atoms have
        // landed goes in one call (a PTX loop, no per-group election); then
        // wait for the next atom.  A group that runs past the ring end reads
        // the guard (a copy of slot 0's atom).
        // whole 4-step groups: the steps past kdim + d meet zero rows of the
        // weight operand (kdim_pad is a whole number of 4-step groups), so the
        // row needs no separately issued tail group
        const int n_full = (nk + 3) >> 2;
        const uint32_t b_lo0 = static_cast<uint32_t>(bvar);
#ifdef MEC_TRACE
        int n_runs = 0;
        long long cyc_fence = 0;
        const long long cyc_setup = clock64() - cyc_row0 - cyc_tempty;
#endif
        if (n_full > 0) {
          // the whole row in one call: the elected lane waits for each atom
          // inside the PTX loop; this warp's ring counters then skip past the
          // last atom the row's full groups need
          if (!no_mma)
            ptx::mma_ts_row_elect<kTF32, kPair>(d_tmem, col, ring0 + ring_cols, ring_cols, b_lo0, b_tile16, p.idesc,
                                         n_full, a, kcl + 2, bkl, ptx::smem_u32(afull), wslot, wphase, avail,
                                         ns);
          const int last = (a + (n_full << (kcl + 2)) - 1) >> bkl;
          while (avail <= last) {
            if (no_mma) ptx::mbar_wait(&afull[wslot], wphase);
            if (++wslot == ns) {
              wslot = 0;
              wphase ^= 1u;
            }
            ++avail;
            ++aseq;
          }
          col += static_cast<uint32_t>(n_full * 32);
          while (col >= ring0 + ring_cols) col -= ring_cols;
          if (no_mma) ptx::tc_fence_after();
        }
#ifdef MEC_TRACE
        const long long c_loop_end = clock64();
#endif
#ifdef MEC_TRACE
        const long long cc0 = clock64();
#endif
        if constexpr (kPair) ptx::mma_commit_pair_elect(&tfull[acc], 0x3);  // both CTAs' epilogues
        else ptx::mma_commit_elect(&tfull[acc]);
#ifdef MEC_TRACE
        const long long cyc_commit = clock64() - cc0;
#endif
        if (lane == 0 && mi == 0 && !(p.dbg & 16)) SW_TRACE(static_cast<uint32_t>(r), 7);
#ifdef MEC_TRACE
        if (lane == 0 && sw_tr != nullptr && blockIdx.x < 160 && r < 256) {
          unsigned long long* e = sw_tr + (static_cast<size_t>(blockIdx.x) * 512 + 256 + r) * 8;
          e[0] = static_cast<unsigned long long>(cyc_tempty) + 1;
          e[1] = static_cast<unsigned long long>(cyc_wait) + 1;
          e[2] = static_cast<unsigned long long>(cyc_issue) + 1;
          e[3] = static_cast<unsigned long long>(clock64() - cyc_row0) + 1;
          e[4] = static_cast<unsigned long long>(cyc_commit) + 1;
          e[5] = static_cast<unsigned long long>(n_runs) + 1;
          e[6] = static_cast<unsigned long long>(cyc_setup) + 1;
          e[7] = static_cast<unsigned long long>(cc0 - c_loop_end) + 1;  // tail
          e[5] = static_cast<unsigned long long>(c_loop_end - cyc_row0 - cyc_tempty - cyc_setup) + 1;  // run loop
        }
#endif
        __syncwarp();
      }
      skip_to(it.n_a);  // atoms no row of this issuer needs: never waited for
      q += static_cast<uint32_t>(it.nrows);
    }
  } else if (warp == 1 || warp == kSwMma2Warp) {
    // (second issuer not used for this problem; pair mode: the peer CTA issues nothing)
  } else if (warp < kSwFirstEpiWarp) {
    // ===================== copiers: smem atom -> TMEM ring =====================
    const int quarter = warp & 3;
    const uint32_t cgroup = static_cast<uint32_t>((warp - kSwFirstCopyWarp) >> 2);  // atoms cseq = cgroup mod groups
    const int m = 32 * quarter + lane;  // tile row = TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(32 * quarter) << 16;
    const uint32_t a_smem = ptx::smem_u32(smemA) + static_cast<uint32_t>(m * kTileKBytes);
    const uint32_t sw = static_cast<uint32_t>(m & 7);
    uint32_t cseq = 0;
    uint32_t q = 0;  // global number of the item's row 0
    // running ring positions (no divisions on this latency-critical path)
    int stage = 0, slot = 0;
    uint32_t sphase = 0;
    const uint32_t afull0 = kPair ? ptx::mapa_shared(ptx::smem_u32(afull), 0) : 0u;  // the leader's ring barriers
    for (int64_t t = t_begin; t < p.n_items; t += t_step) {
      const SwItem it = sw_decode(p, t, kPair, rank);
      const uint32_t jstart = cseq;  // the item's atom 0
      // last row whose window starts at or before atom jj (jj increasing):
      // fr, and fo = the first element of row fr + 1
      int fr = 0, fo = it.off0 + p.shift;
      for (int i = 0; i < it.n_a; ++i, ++cseq) {
        if (kSwCopyGroups > 1 && cseq % kSwCopyGroups != cgroup) {  // another group's atom
          if (++stage == S) {
            stage = 0;
            sphase ^= 1u;
          }
          if (++slot == p.ns) slot = 0;
          continue;
        }
        if (p.backoff_ns) ptx::mbar_wait_backoff(&full[stage], sphase, p.backoff_ns);
        else ptx::mbar_wait(&full[stage], sphase);
        if (warp == kSwFirstCopyWarp && lane == 0) SW_TRACE(cseq, 1);
        uint32_t r[32];
        const uint32_t src = a_smem + static_cast<uint32_t>(stage * kSwAtomBytes);
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // 128-byte swizzle: 16-byte chunk c of row m at c ^ (m mod 8)
          const uint4 x = ptx::ld_shared_v4(src + ((static_cast<uint32_t>(c) ^ sw) << 4));
          r[4 * c] = x.x;
          r[4 * c + 1] = x.y;
          r[4 * c + 2] = x.z;
          r[4 * c + 3] = x.w;
        }
        // the atom is in registers: its shared-memory stage can be refilled now
        // (the arrive's release orders the loads before the next TMA write)
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[stage]);
        if (cseq >= static_cast<uint32_t>(p.ns)) {
          // the slot's previous atom J = cseq - ns is free once the last row
          // reading it completed: in this item row r_max = the last row whose
          // window starts at or before atom J; an atom of an earlier item is
          // free once that item's last row completed
          const uint32_t J = cseq - static_cast<uint32_t>(p.ns);
          uint32_t g_free;
          if (J >= jstart) {
            const int jend = ((static_cast<int>(J - jstart) + 1) << p.bk_log2) - 1;  // last element of atom J
            while (fr + 1 < it.nrows && fo <= jend) {
              ++fr;
              fo += p.shift;
            }
            g_free = q + static_cast<uint32_t>(fr);
          } else {
            g_free = q - 1u;
          }
          // rows of one parity complete in order (one accumulator, one
          // issuer per parity when two issue): rows g_free and g_free - 1
          // cover every earlier row of both parities
          // (one epilogue group when n_acc = 1: its counter covers every row)
          const uint32_t ngl = static_cast<uint32_t>(p.n_acc - 1);  // log2(n_acc), n_acc = 1 or 2
          const uint32_t want = (g_free >> ngl) + 1u;
          while (ptx::ld_acquire_shared_u32(ptx::smem_u32(&rows_done[g_free & ngl])) < want) {
            if (p.backoff_ns) __nanosleep(p.backoff_ns);
          }
          if (g_free > 0 && ngl == 1) {
            const uint32_t g2 = g_free - 1u, want2 = (g2 >> 1) + 1u;
            while (ptx::ld_acquire_shared_u32(ptx::smem_u32(&rows_done[g2 & 1u])) < want2) {
              if (p.backoff_ns) __nanosleep(p.backoff_ns);
            }
          }
        }
        ptx::tc_fence_after();
        if (warp == kSwFirstCopyWarp && lane == 0) SW_TRACE(cseq, 2);
        if (!(p.dbg & 4)) ptx::tmem_st_32x32b_x32(tmem_base + lane_base + p.a_col0 + static_cast<uint32_t>(slot * 32), r);
        if (slot == 0 && !(p.dbg & 4))  // guard: a K group running past the ring end reads it
          ptx::tmem_st_32x32b_x32(tmem_base + lane_base + p.guard_col, r);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair) ptx::mbar_arrive_cluster(afull0 + static_cast<uint32_t>(slot) * 8u);
          else ptx::mbar_arrive(&afull[slot]);
        }
        if (warp == kSwFirstCopyWarp && lane == 0) SW_TRACE(cseq, 3);
        if (++stage == S) {
          stage = 0;
          sphase ^= 1u;
        }
        if (++slot == p.ns) slot = 0;
      }
      q += static_cast<uint32_t>(it.nrows);
    }
  } else {
    // ===================== epilogue (two groups of 4 warps, alternate rows) =====================
    const int quarter = warp & 3;
    const int group = (warp - kSwFirstEpiWarp) >> 2;
    unsigned char* const stg_gen = smemE + static_cast<size_t>(warp - kSwFirstEpiWarp) * p.stage_out_bytes;
    const uint32_t stg = ptx::smem_u32(stg_gen);
    const uint32_t lane_base = static_cast<uint32_t>(32 * quarter) << 16;
    uint32_t q = 0;
    const uint32_t tempty0 = kPair ? ptx::mapa_shared(ptx::smem_u32(tempty), 0) : 0u;
    for (int64_t t = t_begin; t < p.n_items; t += t_step) {
      const SwItem it = sw_decode(p, t, kPair, rank);
      for (int r = 0; r < it.nrows; ++r) {
        const uint32_t qr = q + static_cast<uint32_t>(r);
        const uint32_t al = static_cast<uint32_t>(p.n_acc - 1);  // log2(n_acc), n_acc = 1 or 2
        const int acc = static_cast<int>(qr & al);
        if (kSwEpiGroups > 1 && acc != group) continue;  // (n_acc = 1 or one group: group 0 takes every row)
        if (p.backoff_ns) ptx::mbar_wait_backoff(&tfull[acc], (qr >> al) & 1u, p.backoff_ns);
        else ptx::mbar_wait(&tfull[acc], (qr >> al) & 1u);
        ptx::tc_fence_after();
        // row qr's MMAs are complete: its A atoms may be overwritten
        if (lane == 0 && ((warp - kSwFirstEpiWarp) & 3) == 0)
          ptx::st_release_shared_u32(ptx::smem_u32(&rows_done[acc]), (qr >> al) + 1u);
        sw_store_row<kTF32>(p, &tmO, it.h0 + r, it.mt, it.g, quarter, lane,
                            tmem_base + lane_base + static_cast<uint32_t>(acc * p.bn), stg, stg_gen, &tempty[acc],
                            it.valid, kPair ? tempty0 + static_cast<uint32_t>(acc) * 8u : 0u);
      }
      q += static_cast<uint32_t>(it.nrows);
    }
    if (lane == 0) ptx::bulk_wait_group<0>();
    if (lane == 0 && warp == kSwFirstEpiWarp) SW_TRACE(511u, 4);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kPair) ptx::cluster_sync();  // no MMA, commit or remote arrive of the pair in flight
  if (threadIdx.x == 0) SW_TRACE(511u, 5);
  if (warp == 1) {
    ptx::tc_fence_after();
    if constexpr (kPair) ptx::tmem_dealloc_pair(tmem_base, 512);
    else ptx::tmem_dealloc(tmem_base, 512);
  }
}

constexpr size_t kSwSmemBudget = 222 * 1024;
constexpr int kSwMaxStages = 8;  // the barrier block holds 8 full + 8 empty barriers

// epilogue pass width in bytes of an output row (128, 64 or 32, dividing
// bn elt); MEC_SWEEP_EPI_BYTES caps it (experiments: less staging, more stages)
int sweep_epi_row_bytes(const Plan& pl) {
  int row_bytes = 128;
  if (const char* e = getenv("MEC_SWEEP_EPI_BYTES")) row_bytes = std::max(32, std::min(128, atoi(e)));
  while (row_bytes > 32 && (pl.bn * pl.elt) % row_bytes != 0) row_bytes /= 2;
  return row_bytes;
}

// CTA-pair mode of the h-sweep (MEC_SWEEP_PAIR=1 / 0 forces it on / off)
bool sweep_pair_mode(const Plan& pl) {
  if (const char* e = getenv("MEC_SWEEP_PAIR")) return atoi(e) != 0;
  (void)pl;
  return false;
}

int ilog2(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}

}  // namespace

// The sweep's resources for plan pl, or false when it does not apply (then
// the one-window-per-tile kernel runs).
bool sweep_config(const Plan& pl, bool batch_folded, int* n_vres_out, int* n_acc_out, int* ns_out,
                  int* stages_out, bool pair) {
  if (getenv("MEC_SWEEP") && atoi(getenv("MEC_SWEEP")) == 0) return false;
  if (pl.n_tiles_n != 1 || pl.o_h < 2 || pl.shift >= pl.kdim) return false;  // no window overlap: nothing to share
  if (pl.l_cols > (1LL << 30) || pl.o_h * pl.shift > (1LL << 30)) return false;
  const int mvec = 16 / pl.elt;
  int64_t g = pl.shift % mvec, b = mvec;
  while (g) { const int64_t t = b % g; b = g; g = t; }
  const int n_vres = static_cast<int>(mvec / b);  // variants d = (h shift) mod mvec, multiples of gcd(shift, mvec)
  if (n_vres > pl.n_var) return false;
  if (n_vres > 1 && pl.delta_step != b) return false;
  const int kc = 32 / pl.elt;
  // TMEM: n_acc accumulators (rows in flight between MMA and epilogue) and a
  // ring of ns atoms that holds one row's whole window (span atoms) plus
  // look-ahead, and the guard
  // (worst case over the window's start inside an atom and over d)
  int span = 0;
  for (int phi = 0; phi < pl.bk; phi += mvec)
    for (int d = 0; d < mvec; d += static_cast<int>(b)) {
      const int64_t nk = ((pl.kdim + d + kc - 1) / kc + 3) / 4 * 4;
      span = std::max<int>(span, static_cast<int>((phi + nk * kc - 1) / pl.bk) + 1);
    }
  // two accumulators (one per MMA issuer, or double-buffered), else one
  // (k_c = 128: the ring then holds a 10-atom window; rows serialise on it)
  int n_acc = 2;
  int ns = std::min(kSwMaxRing, (512 - kSwGuardCols - ((2 * pl.bn + 31) / 32) * 32) / 32);
  if (ns < span || (getenv("MEC_SWEEP_NACC") && atoi(getenv("MEC_SWEEP_NACC")) == 1)) {  // (env: experiments)
    n_acc = 1;
    ns = std::min(kSwMaxRing, (512 - kSwGuardCols - ((pl.bn + 31) / 32) * 32) / 32);
  }
  if (ns < span) return false;
  int row_bytes = sweep_epi_row_bytes(pl);
  const size_t epi = static_cast<size_t>(kSwEpiWarps) * 32 * row_bytes;
  // (pair mode: each CTA holds bn / 2 rows of the weights)
  const size_t b_res = static_cast<size_t>(n_vres) * (pl.kdim_pad / pl.bk) * (pair ? pl.bn / 2 : pl.bn) * kTileKBytes;
  const size_t fixed = b_res + epi + 66 * 8 + 64;
  if (fixed + 2 * kSwAtomBytes > kSwSmemBudget) return false;
  int stages = static_cast<int>(std::min<size_t>(kSwMaxStages, (kSwSmemBudget - fixed) / kSwAtomBytes));
  if (const char* e = getenv("MEC_SWEEP_STAGES")) stages = std::max(2, std::min(stages, atoi(e)));  // (experiments)
  (void)batch_folded;
  *n_vres_out = n_vres;
  *n_acc_out = n_acc;
  *ns_out = ns;
  *stages_out = stages;
  return true;
}

cudaError_t launch_sweep_gemm(const Plan& pl, const GemmArgs& a, cudaStream_t st, int* launches) {
  int n_vres, n_acc, ns, stages;
  if (a.fused && !fused_eligible(pl)) return cudaErrorNotSupported;
  if (!sweep_config(pl, a.batch_folded, &n_vres, &n_acc, &ns, &stages, false)) return cudaErrorNotSupported;
  // CTA pairs: the 2-SM TS MMA needs N a multiple of 32
  const bool pair = sweep_pair_mode(pl) && pl.bn % 32 == 0;
  if (pair && !sweep_config(pl, a.batch_folded, &n_vres, &n_acc, &ns, &stages, true)) return cudaErrorNotSupported;
  const bool tf32 = pl.dt == MEC_DTYPE_TF32;
  const int out_elt = pl.elt;
  CUtensorMap tmA, tmB, tmO;
  // row tiling: as window_gemm.cu
  // flat batch-folded rows (n o_w + w, 128 per tile, one TMA box per atom)
  // for o_w < 32, and for o_w <= 64 where the window shift is 16-byte aligned
  // (one weight copy): measured C3 GEMM 85.3 -> 79.0 us, cv9 b128 51.4 -> 46.2,
  // while AlexNet conv1's shape (two weight copies) kept image slots (C1 22.5
  // vs 24.8 us; profiles/r2_sweep_flat_rows.txt).  MEC_SWEEP_FLAT64=0: slots.
  const bool flat64 = pl.o_w <= 64 && pl.shift % (16 / pl.elt) == 0 &&
                      !(getenv("MEC_SWEEP_FLAT64") && atoi(getenv("MEC_SWEEP_FLAT64")) == 0);
  const bool flat = !a.fused && a.batch_folded && (pl.o_w < 32 || flat64);
  int slot = 128, ipt = 1;
  if (!flat && pl.o_w <= 128) {
    slot = static_cast<int>((pl.o_w + 31) / 32 * 32);
    if (a.batch_folded) ipt = std::max(1, 128 / slot);
    if (ipt == 1) slot = 128;
  }
  const int64_t rows = flat ? pl.s.i_n * pl.o_w : pl.o_w;
  const int64_t groups = flat ? 1 : (pl.s.i_n + ipt - 1) / ipt;
  const int64_t n_mt = flat ? (rows + kBM - 1) / kBM : (ipt > 1 ? 1 : (pl.o_w + kBM - 1) / kBM);
  if (a.fused) {
    // A: the NHWC input as {i_c, i_w, i_h, i_n}; a box is bk channels x `rows`
    // pixels taken every s_w pixels (elementStrides): one K-atom of the stream
    const uint64_t dims[4] = {static_cast<uint64_t>(pl.s.i_c), static_cast<uint64_t>(pl.src_w),
                              static_cast<uint64_t>(pl.src_h), static_cast<uint64_t>(pl.s.i_n)};
    const uint64_t strides[3] = {static_cast<uint64_t>(pl.s.i_c) * pl.elt,
                                 static_cast<uint64_t>(pl.src_w * pl.s.i_c) * pl.elt,
                                 static_cast<uint64_t>(pl.src_h * pl.src_w * pl.s.i_c) * pl.elt};
    const uint32_t rows_box = static_cast<uint32_t>(ipt > 1 ? slot : kBM);
    const uint32_t box[4] = {static_cast<uint32_t>(pl.bk), rows_box * static_cast<uint32_t>(pl.s_w), 1,
                             static_cast<uint32_t>(ipt)};
    const uint32_t es[4] = {1, static_cast<uint32_t>(pl.s_w), 1, 1};
    cudaError_t e = encode_tiled_strided(&tmA, tf32, 4, a.L, dims, strides, box, es);
    if (e != cudaSuccess) return e;
  } else {  // A: L as {columns, rows, groups} (flat: one group of i_n o_w rows)
    const uint64_t dims[3] = {static_cast<uint64_t>(pl.l_cols), static_cast<uint64_t>(rows),
                              static_cast<uint64_t>(flat ? 1 : pl.s.i_n)};
    const uint64_t strides[2] = {static_cast<uint64_t>(pl.pitch) * pl.elt,
                                 static_cast<uint64_t>(pl.pitch) * pl.elt * rows};
    const uint32_t box[3] = {static_cast<uint32_t>(pl.bk), static_cast<uint32_t>(ipt > 1 ? slot : kBM),
                             static_cast<uint32_t>(ipt)};
    cudaError_t e = encode_tiled(&tmA, tf32, 3, a.L, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  {  // B: Kt, n_var x kc_pad rows of kdim_pad (K-major)
    const uint64_t dims[2] = {static_cast<uint64_t>(pl.kdim_pad), static_cast<uint64_t>(pl.n_var * pl.kc_pad)};
    const uint64_t strides[1] = {static_cast<uint64_t>(pl.kdim_pad) * pl.elt};
    const uint32_t box[2] = {static_cast<uint32_t>(pl.bk), static_cast<uint32_t>(pair ? pl.bn / 2 : pl.bn)};
    cudaError_t e = encode_tiled(&tmB, tf32, 2, a.Kt, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  SweepParams p{};
  p.O = a.O;
  p.fused = a.fused;
  p.kwc = static_cast<int>(pl.s.k_w * pl.s.i_c);
  p.i_c = static_cast<int>(pl.s.i_c);
  p.s_w = pl.s_w;
  p.pad_h = pl.pad_h;
  p.pad_w = pl.pad_w;
  p.o_h = pl.o_h;
  p.o_w = pl.o_w;
  p.i_n = pl.s.i_n;
  p.k_c = pl.s.k_c;
  p.flat = flat;
  p.ipt = ipt;
  p.slot = slot;
  p.rows = rows;
  p.groups = groups;
  p.n_mt = n_mt;
  p.shift = static_cast<int>(pl.shift);
  p.kdim = static_cast<int>(pl.kdim);
  p.bk = pl.bk;
  p.bk_log2 = ilog2(pl.bk);
  p.kchunk_log2 = pl.elt == 2 ? 4 : 3;
  p.mvec = 16 / pl.elt;
  p.avec = pl.avec;
  p.ds_log2 = ilog2(pl.delta_step);
  p.nb_atoms = static_cast<int>(pl.kdim_pad / pl.bk);
  p.n_vres = n_vres;
  p.kc_pad = pl.kc_pad;
  p.bn = pl.bn;
  p.stages = stages;
  p.ns = ns;
  p.n_acc = n_acc;
  p.a_col0 = static_cast<uint32_t>(((n_acc * pl.bn + 31) / 32) * 32);
  p.guard_col = p.a_col0 + static_cast<uint32_t>(32 * ns);
  p.idesc = ptx::instr_desc(tf32, pair ? 2 * kBM : kBM, pl.bn);
  p.col_shift = pl.elt == 2 ? 1 : 0;
  p.out_hnwc = a.out_hnwc;
  p.dbg = getenv("MEC_SWEEP_DBG") ? atoi(getenv("MEC_SWEEP_DBG")) : 0;
  // (measured: C2 GEMM 309 -> 307.5 us, cv7 b128 232.7 -> 230.3 us, C3 equal;
  // profiles/r2_sweep_reverse.txt.  MEC_SWEEP_REV=0: forward order)
  p.reverse = !a.fused && !(getenv("MEC_SWEEP_REV") && atoi(getenv("MEC_SWEEP_REV")) == 0);
  // two issuers need every atom read by both issuers' rows (windows of rows
  // h and h + 2 overlap), else an issuer could lag a slot by two fills
  // (measured: 2 issuers win where the accumulators are 64 columns -- C2
  // 434->397 us, C3 127->117 us, cv3 106->95 us, cv7 255->250 us -- and lose
  // ~4-7% at k_c = 96, C1 / cv1, whose TMEM ring has 2 slots fewer)
  // cp mode (MEC_SWEEP_CP=1 / 0): the MMA thread copies the atoms into TMEM
  // itself (tcgen05.cp), one issuer; not with CTA pairs (one cta_group per kernel)
  p.cp = !pair && getenv("MEC_SWEEP_CP") && atoi(getenv("MEC_SWEEP_CP")) != 0;
  p.n_iss = (2 * pl.shift < pl.kdim && pl.bn <= 64 && n_acc == 2) ? 2 : 1;
  if (const char* e = getenv("MEC_SWEEP_ISSUERS"))  // (experiments; 2 needs 2 shift < kdim, 2 accumulators)
    p.n_iss = (atoi(e) >= 2 && 2 * pl.shift < pl.kdim && n_acc == 2) ? 2 : 1;
  if (p.cp) p.n_iss = 1;
  p.backoff_ns = getenv("MEC_SWEEP_BACKOFF") ? static_cast<uint32_t>(atoi(getenv("MEC_SWEEP_BACKOFF"))) : 0u;
  // epilogue: pass width = 128 / 64 / 32 bytes per row, dividing bn
  const int row_bytes = sweep_epi_row_bytes(pl);
  p.pw = row_bytes / out_elt;
  p.n_pass = pl.bn / p.pw;
  p.tma_store = ((pl.s.k_c * out_elt) % 16 == 0) && (reinterpret_cast<uintptr_t>(a.O) % 16 == 0) &&
                pl.s.k_c % p.pw == 0;
  p.stage_out_bytes = static_cast<uint32_t>(32 * row_bytes);
  if (p.tma_store) {
    cudaError_t e;
    if (a.out_hnwc && flat) {  // O_hnwc as {k_c, i_n o_w, o_h}
      const uint64_t dims[3] = {static_cast<uint64_t>(pl.s.k_c), static_cast<uint64_t>(pl.s.i_n * pl.o_w),
                                static_cast<uint64_t>(pl.o_h)};
      const uint64_t strides[2] = {static_cast<uint64_t>(pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.s.i_n * pl.o_w * pl.s.k_c) * out_elt};
      const uint32_t box[3] = {static_cast<uint32_t>(p.pw), 32, 1};
      e = encode_tiled_swz(&tmO, tf32, 3, a.O, dims, strides, box, row_bytes);
    } else if (a.out_hnwc) {  // O_hnwc as {k_c, o_w, i_n, o_h}
      const uint64_t dims[4] = {static_cast<uint64_t>(pl.s.k_c), static_cast<uint64_t>(pl.o_w),
                                static_cast<uint64_t>(pl.s.i_n), static_cast<uint64_t>(pl.o_h)};
      const uint64_t strides[3] = {static_cast<uint64_t>(pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.o_w * pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.s.i_n * pl.o_w * pl.s.k_c) * out_elt};
      const uint32_t box[4] = {static_cast<uint32_t>(p.pw), 32, 1, 1};
      e = encode_tiled_swz(&tmO, tf32, 4, a.O, dims, strides, box, row_bytes);
    } else {  // O as {k_c, o_w, o_h, i_n}
      const uint64_t dims[4] = {static_cast<uint64_t>(pl.s.k_c), static_cast<uint64_t>(pl.o_w),
                                static_cast<uint64_t>(pl.o_h), static_cast<uint64_t>(pl.s.i_n)};
      const uint64_t strides[3] = {static_cast<uint64_t>(pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.o_w * pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.o_h * pl.o_w * pl.s.k_c) * out_elt};
      const uint32_t box[4] = {static_cast<uint32_t>(p.pw), 32, 1, 1};
      e = encode_tiled_swz(&tmO, tf32, 4, a.O, dims, strides, box, row_bytes);
    }
    if (e != cudaSuccess) return e;
  } else {
    std::memset(&tmO, 0, sizeof(tmO));
  }

  // h-chunk size H: minimise (waves) x (bytes one item moves: its stream of
  // atoms, its O rows and a fixed pipeline fill), ties to fewer items
  const int64_t tiles = n_mt * groups;
  p.n_tiles = tiles;
  // pair mode: items are (h chunk, pair of CTA tiles), one per pair of SMs
  const int64_t work_tiles = pair ? (tiles + 1) / 2 : tiles;
  const int sms = pair ? std::max(1, num_sms() / 2) : num_sms();
  const double o_row_bytes = static_cast<double>(kBM) * pl.bn * out_elt;
  double best = 1e300;
  int64_t best_H = pl.o_h;
  int64_t best_n = 1;
  for (int64_t n_hc = 1; n_hc <= pl.o_h; ++n_hc) {
    const int64_t H = (pl.o_h + n_hc - 1) / n_hc;  // the largest chunk
    const int64_t items = n_hc * work_tiles;
    const int64_t waves = (items + sms - 1) / sms;
    const double atoms = static_cast<double>((H - 1) * pl.shift + pl.kdim + pl.avec) / pl.bk + 1.0;
    const double cost = static_cast<double>(waves) * (atoms * kSwAtomBytes + H * o_row_bytes + 4.0 * kSwAtomBytes);
    if (cost < best * 0.999) {
      best = cost;
      best_H = H;
      best_n = n_hc;
    }
  }
  // balanced split (not CTA pairs): one CTA per SM, each the same number of
  // (tile, h) rows, cut at tile boundaries, where the chunked items above
  // leave SMs idle (C3, cv1-cv3, cv9 at b128: 128 tiles of one chunk for 148
  // SMs) and the cost model (a CTA's pieces' streams + rows + fills) agrees.
  // Measured (profiles/r2_sweep_balanced.txt): C3 GEMM 92.3 -> 86.2 us, cv3
  // b128 90.5 -> 82.5; C1 (two fills per ~6-row CTA) and C2 (chip-wide
  // DRAM-bound, every SM already busy) gain nothing and keep the chunks.
  bool balanced = false;
  int64_t bal_G = 0, bal_J = 0;
  const int64_t R = tiles * pl.o_h;
  if (!pair && R >= sms && best_n * work_tiles < sms) {
    bal_G = sms;
    const int64_t per = (R + bal_G - 1) / bal_G;
    bal_J = (per + pl.o_h - 1) / pl.o_h + 1;
    double worst = 0.0;
    for (int64_t c = 0; c < bal_G; ++c) {
      const int64_t s0 = c * R / bal_G, e0 = (c + 1) * R / bal_G;
      double cost = 0.0;
      for (int64_t pos = s0; pos < e0;) {
        const int64_t end = std::min(e0, (pos / pl.o_h + 1) * pl.o_h);
        const int64_t H = end - pos;
        const double atoms = static_cast<double>((H - 1) * pl.shift + pl.kdim + pl.avec) / pl.bk + 1.0;
        cost += atoms * kSwAtomBytes + H * o_row_bytes + 4.0 * kSwAtomBytes;
        pos = end;
      }
      worst = std::max(worst, cost);
    }
    balanced = worst < best * 0.999;
    if (const char* e = getenv("MEC_SWEEP_BALANCED")) balanced = atoi(e) != 0;
  }
  if (const char* e = getenv("MEC_SWEEP_H")) {
    best_H = std::max<int64_t>(1, std::min<int64_t>(pl.o_h, atoi(e)));
    best_n = (pl.o_h + best_H - 1) / best_H;
    balanced = false;
  }
  if (work_tiles * pl.o_h >= (1LL << 31) || pl.s.i_n * pl.o_w >= (1LL << 31))
    return cudaErrorNotSupported;  // (the kernel's item and row indices are 32-bit)
  p.H = static_cast<int>(best_H);
  p.n_hc = best_n;
  p.n_items = p.n_hc * work_tiles;
  if (balanced) {
    p.bal_R = R;
    p.bal_G = static_cast<int>(bal_G);
    p.bal_J = static_cast<int>(bal_J);
    p.n_items = bal_G * bal_J;
    p.H = static_cast<int>(std::min<int64_t>(pl.o_h, (R + bal_G - 1) / bal_G));
  }

  const size_t b_res = static_cast<size_t>(n_vres) * p.nb_atoms * (pair ? pl.bn / 2 : pl.bn) * kTileKBytes;
  const size_t smem = kSmemAlign + static_cast<size_t>(stages) * kSwAtomBytes + b_res +
                      static_cast<size_t>(kSwEpiWarps) * p.stage_out_bytes + 66 * 8 + 16;
  if (smem > kSwSmemBudget + kSmemAlign + 2048) return cudaErrorInvalidConfiguration;
  auto kern = tf32 ? (pair ? sweep_gemm_kernel<true, true> : sweep_gemm_kernel<true, false>)
                   : (pair ? sweep_gemm_kernel<false, true> : sweep_gemm_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kSwThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = pair ? attr + 1 : attr;
  cfg.numAttrs = 0;
  int64_t grid = std::min<int64_t>(p.n_items, sms);
  if (pair) {
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(static_cast<unsigned>(2 * sms));
    int max_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
      cudaGetLastError();
      max_clusters = sms;
    }
    grid = 2 * std::min<int64_t>(p.n_items, max_clusters);
    // the PDL attribute next to the cluster one
    if (!getenv("MEC_NO_PDL")) {
      cfg.attrs = attr;
      cfg.numAttrs = 2;
    }
  } else if (!getenv("MEC_NO_PDL")) {
    cfg.numAttrs = 1;
  }
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmO, p);
  if (e != cudaSuccess) return e;
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace mec
