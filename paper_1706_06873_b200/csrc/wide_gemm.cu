// wide_gemm.cu -- the window GEMMs of the tensor-bound layers on CTA pairs
// (tcgen05 cta_group::2, M = 256), with split-K across pairs (sm_100a).
//
// Paper: Solution A (batch-folded, Alg.2 l.10-12):
//   O[h, 0:i_n o_w k_c] = L[0:i_n o_w, s_h k_w i_c h : + k_h k_w i_c] x K
// i.e. per output row h one GEMM of an overlapping window of L (a sub-matrix
// "specified by providing a pointer to the initial element and ld")
// times K.  P:211-213: on GPUs the size of those sub-matrices decides the
// speed.  For the deep layers of Table 2 (cv5, cv6, cv11, cv12: o_w <= 20,
// k_h k_w i_c >= 2304, k_c >= 256) the window GEMMs are tensor-bound (SURVEY
// 8(d): 510-857 F/B against a 251 F/B ridge), and two things limit the
// one-window kernel (window_gemm.cu) there:
//   * operand traffic from L2: an M = 128, N = 256 tile streams 48 KB of A and
//     B per 128-byte K atom, 96 B per tensor-core cycle per SM, more than L2
//     delivers.  Here two CTAs on the two SMs of a TPC issue the MMAs as one
//     pair (cta_group::2): M = 256, each CTA loads its 128 rows of A and half
//     of B's N columns, 64 B per cycle per SM.
//   * too few tiles: cv12 at batch 128 has 5 output rows x 640 folded rows
//     x 512 channels = 30 pair tiles for 74 SM pairs.  The K loop of a tile is
//     split into S ranges (split-K) run by different pairs.  The ranges then
//     exchange partials (a reduce-scatter through L2): range k owns 1/S of
//     the tile's output columns, writes its fp32 partial of the other columns
//     to a workspace slot, counts itself in on a per-(tile, 32-row block)
//     counter, waits for the other ranges' counts, and sums its own columns'
//     S partials IN RANGE ORDER (so the result does not depend on which range
//     finished first) before storing O.  Measured on B200 (cv12 b128, S = 2):
//     GEMM 31.1 us with the earlier last-arriver-sums-everything scheme, 27.8
//     with the exchange, 24.6 with no partial traffic at all.
//
// The windows are read in place from L with TMA (2-D map {i_h k_w i_c, i_n
// o_w}, the box at column h s_h k_w i_c rounded down to the 32-byte box
// alignment, weight copy v absorbing the remainder, as in window_gemm.cu), so
// no im2col buffer exists.  O is stored in n-h-w-c (Solution A's permutation,
// Alg.2 l.17-19, applied at store time).
//
// Kernel structure (persistent, one CTA pair per TPC, 10 warps per CTA):
//   warp 0     TMA producer (both CTAs): per K atom this CTA's 128 rows of the
//              A window (16 KB) and its N/2 rows of Kt, completing on the
//              LEADER's full barrier (one expect_tx covers both CTAs).
//   warp 1     TMEM allocator (both CTAs, cta_group::2) and, in the leader,
//              the MMA issuer: 4 MMAs (M 256, N bn, K 32 bytes) per atom,
//              commits multicast to both CTAs' barriers.
//   warps 2-9  two epilogue groups (alternate units = the 2 TMEM accumulators):
//              tcgen05.ld -> [split-K partial / reduction] -> bf16 or fp32 ->
//              swizzled smem staging -> coalesced 16-byte stores of O rows.
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

namespace mec {
namespace {

constexpr int kWideThreads = 64 + 2 * 128;
constexpr int kPairM = 2 * kBM;                 // 256 rows per pair tile
constexpr int kAtomA = kBM * kTileKBytes;       // 16 KB: this CTA's 128 rows of one K atom
constexpr uint32_t kStageOut = 32 * 128;        // epilogue staging: 32 rows x 128 bytes per warp
constexpr size_t kWideSmemBudget = 227 * 1024;  // dynamic smem per CTA (sm_100)
constexpr int kMaxSplit = 8;

struct WideParams {
  void* O;
  float* part;     // split-K partial slots (S > 1)
  uint32_t* cnt;   // split-K arrival counters, zero on entry
  int64_t o_h, o_w, i_n, k_c;
  int64_t rows;    // i_n o_w (flat batch-folded rows)
  int64_t n_mt;    // ceil(rows / 256)
  int n_ng;        // N groups: n_tiles_n / n_sub
  int bn;          // MMA N (<= 256)
  int n_sub;       // N tiles per unit (1, or 2: N = 2 bn, both TMEM halves, no double buffer)
  int n_var, avec, delta_step;
  int64_t shift, kc_pad;
  int bk;          // K-atom width in elements (64 bf16 / 32 fp32)
  int n_atoms;     // K atoms per window
  int S, apk;      // split count, atoms per split
  int64_t n_tiles, n_units;
  int64_t g_full;  // unit groups run as whole tiles before the split ones (0: every tile split S ways)
  // pairs per cluster sharing one multicast of the weights (mc, 1 or 2): a
  // cluster works on `mc` (h, 256-row) tiles of the same N group and K range
  int mc;
  int64_t n_hm, n_groups;  // (h, 256-row tile) combos; unit groups = ceil(n_hm / mc) n_ng S
  int stages;
  uint32_t stage_bytes, a_bytes, b_half_bytes;
  uint32_t idesc;
  // weights read straight from K (MN-major B): each CTA's N/2
  // columns come as b_chunks TMA boxes of chunk_n columns x bk K rows
  bool b_mn;
  int b_chunks, chunk_n;
  uint32_t b_chunk_bytes, b_kstep16;
  int dbg;  // (timing experiments, MEC_WIDE_DBG: 1 skip the partial reads, 2 skip the partial writes)
};

struct Unit {
  int64_t h, mt, tile;
  int ng, ks, a0, a1;
  int nsplit;  // K ranges of this unit's tile (1: whole tile; p.S: a split tile)
  bool valid;  // false: a cluster's extra pair past the last tile (computes, stores nothing)
};

// unit group G (one per cluster iteration) -> the unit of pair pp of the cluster
__device__ __forceinline__ Unit decode_unit(const WideParams& p, int64_t G64, int pp) {
  Unit c;
  // 32-bit index math (unit groups, tiles and h all fit, launch_wide_gemm):
  // every role decodes each unit before its first atom
  const uint32_t G = static_cast<uint32_t>(G64), g_full = static_cast<uint32_t>(p.g_full);
  const uint32_t S = static_cast<uint32_t>(p.S), n_ng = static_cast<uint32_t>(p.n_ng);
  // the first g_full unit groups are whole tiles (hybrid split: whole waves
  // of unsplit tiles, then the last partial wave's tiles in p.S ranges)
  uint32_t g2;
  if (G < g_full) {
    g2 = G;
    c.ks = 0;
    c.nsplit = 1;
  } else {
    const uint32_t gt = (G - g_full) / S;
    c.ks = static_cast<int>(G - g_full - gt * S);
    g2 = g_full + gt;
    c.nsplit = p.S;
  }
  // K range fastest, then the N group, then the (h, 256-row tile) combo: the
  // pairs in flight share A windows (same rows, neighbouring h) in L2
  const uint32_t hmg = g2 / n_ng;
  c.ng = static_cast<int>(g2 - hmg * n_ng);
  uint32_t hm = hmg * static_cast<uint32_t>(p.mc) + static_cast<uint32_t>(pp);
  const uint32_t n_hm = static_cast<uint32_t>(p.n_hm), o_h = static_cast<uint32_t>(p.o_h);
  c.valid = hm < n_hm;
  if (!c.valid) hm = n_hm - 1;  // (loads a real tile; the epilogue stores nothing)
  c.mt = hm / o_h;
  c.h = hm - static_cast<uint32_t>(c.mt) * o_h;
  c.tile = static_cast<int64_t>(hm) * p.n_ng + c.ng;
  c.a0 = c.nsplit == 1 ? 0 : c.ks * p.apk;
  c.a1 = c.nsplit == 1 ? p.n_atoms : min(p.n_atoms, c.a0 + p.apk);
  return c;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <bool kTF32, int kMc>
__global__ void __launch_bounds__(kWideThreads, 1)
    wide_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const WideParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + kSmemAlign - 1) & ~uintptr_t(kSmemAlign - 1));
  const int S = p.stages;
  unsigned char* stg_base = smem + static_cast<size_t>(S) * p.stage_bytes;  // 8 x 4 KB epilogue staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg_base + 8 * kStageOut);
  uint64_t* full = bars;            // [S] leader: A+B of both CTAs landed
  uint64_t* empty = bars + S;       // [S] each CTA: the stage's MMAs are done
  uint64_t* tfull = bars + 2 * S;   // [2] each CTA: accumulator ready
  uint64_t* tempty = bars + 2 * S + 2;  // [2] leader: both CTAs' epilogue warps drained it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  // cluster = kMc CTA pairs (ranks 2 pp, 2 pp + 1); rank = this CTA's role in its pair
  const uint32_t crank = ptx::cluster_ctarank();
  const uint32_t rank = crank & 1u;
  const int pp = static_cast<int>(crank >> 1);
  const uint32_t leader_rank = crank & ~1u;
  const bool leader = rank == 0;
  const int64_t pair = ptx::cluster_id_x();       // cluster index (unit groups G = pair + k n_pairs)
  const int64_t n_pairs = ptx::nclusters_x();

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], kMc);  // every pair's MMAs release the stage (multicast commits)
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      // 4 epilogue warps x 2 CTAs per accumulator; with n_sub = 2 both groups drain it
      ptx::mbar_init(&tempty[i], 8 * p.n_sub);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();      // the allocator's write of tmem_slot before any read (a CTA barrier racecheck models)
  ptx::cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      const uint64_t hintA = ptx::policy_evict_normal();
      const uint64_t hintB = ptx::policy_evict_last();
      ptx::griddep_wait();  // L and Kt come from the preceding (lowering) kernel
      const uint32_t full0 = ptx::mapa_shared(ptx::smem_u32(full), leader_rank);
      // the weights of the cluster's N group: pair 0 loads each CTA role's half
      // and multicasts it to that role in every pair
      const uint16_t b_mask = static_cast<uint16_t>((kMc == 2 ? 0x5u : 0x1u) << rank);
      const uint32_t tx = 2 * (p.a_bytes + static_cast<uint32_t>(p.n_sub) * p.b_half_bytes);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = pair; u < p.n_groups; u += n_pairs) {
        const Unit c = decode_unit(p, u, pp);
        const int64_t xw = c.h * p.shift;
        const int32_t x0 = static_cast<int32_t>(xw - xw % p.avec);
        const int v = static_cast<int>((xw % p.avec) / p.delta_step);
        const int32_t y0 = static_cast<int32_t>(c.mt * kPairM + rank * kBM);
        const int32_t brow = static_cast<int32_t>(v * p.kc_pad + c.ng * p.n_sub * p.bn + rank * (p.bn / 2));
        // MN-major: B rows = K_mat rows of the box's columns, shifted by the
        // window's delta (negative rows / rows past kdim: TMA zero fill)
        const int32_t bcol = static_cast<int32_t>(c.ng * p.n_sub * p.bn + rank * (p.bn / 2));
        const int32_t bdelta = static_cast<int32_t>(v * p.delta_step);
        for (int a = c.a0; a < c.a1; ++a) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], tx);
          unsigned char* dA = smem + static_cast<size_t>(stage) * p.stage_bytes;
          const uint32_t fb = full0 + static_cast<uint32_t>(stage) * 8u;
          ptx::tma_load_2d_pair(dA, &tmA, fb, x0 + a * p.bk, y0, hintA);
          if (p.b_mn) {
            for (int sb = 0; sb < p.n_sub; ++sb)
              for (int cb = 0; cb < p.b_chunks; ++cb)
                ptx::tma_load_2d_pair(dA + p.a_bytes + sb * p.b_half_bytes + cb * p.b_chunk_bytes, &tmB, fb,
                                      bcol + sb * p.bn + cb * p.chunk_n, a * p.bk - bdelta, hintB);
          } else if (kMc == 1) {
            for (int sb = 0; sb < p.n_sub; ++sb)
              ptx::tma_load_2d_pair(dA + p.a_bytes + sb * p.b_half_bytes, &tmB, fb, a * p.bk, brow + sb * p.bn, hintB);
          } else if (pp == 0) {
            for (int sb = 0; sb < p.n_sub; ++sb)
              ptx::tma_load_2d_pair_mc(dA + p.a_bytes + sb * p.b_half_bytes, &tmB,
                                       ptx::smem_u32(&full[stage]), b_mask, a * p.bk, brow + sb * p.bn, hintB);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (pair leader) =====================
    if (leader) {
      const uint64_t desc0 = ptx::smem_desc_sw128(ptx::smem_u32(smem));
      const uint64_t bmn0 = ptx::smem_desc_sw128_mn(ptx::smem_u32(smem) + p.a_bytes, p.b_chunk_bytes);
      const uint32_t a_to_b = p.a_bytes >> 4, b_to_b = p.b_half_bytes >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int64_t i = 0;
      for (int64_t u = pair; u < p.n_groups; u += n_pairs, ++i) {
        const Unit c = decode_unit(p, u, pp);
        // n_sub = 1: accumulators alternate (i & 1); n_sub = 2: one set of 2 x bn columns
        const int acc = p.n_sub == 1 ? static_cast<int>(i & 1) : 0;
        const int64_t use = p.n_sub == 1 ? (i >> 1) : i;  // uses of this accumulator so far
        ptx::mbar_wait(&tempty[acc], (static_cast<uint32_t>(use) & 1u) ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * p.bn);
        for (int a = c.a0; a < c.a1; ++a) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t soff = static_cast<uint32_t>(stage) * p.stage_bytes >> 4;
          const uint64_t ad = desc0 + soff;
          if (p.b_mn) {
            const uint64_t bd = bmn0 + soff;
            ptx::mma_ss_atom_pair_bstep_elect<kTF32>(d, ad, bd, p.b_kstep16, p.idesc, a != c.a0 ? 1u : 0u);
            if (p.n_sub == 2)
              ptx::mma_ss_atom_pair_bstep_elect<kTF32>(d + static_cast<uint32_t>(p.bn), ad, bd + b_to_b,
                                                       p.b_kstep16, p.idesc, a != c.a0 ? 1u : 0u);
          } else {
            ptx::mma_ss_atom_pair_elect<kTF32>(d, ad, ad + a_to_b, p.idesc, a != c.a0 ? 1u : 0u);
            if (p.n_sub == 2)
              ptx::mma_ss_atom_pair_elect<kTF32>(d + static_cast<uint32_t>(p.bn), ad, ad + a_to_b + b_to_b, p.idesc,
                                                 a != c.a0 ? 1u : 0u);
          }
          // the stage is free in every CTA of the cluster once every pair's MMAs read it
          ptx::mma_commit_pair_elect(&empty[stage], static_cast<uint16_t>(kMc == 2 ? 0xF : 0x3));
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit_pair_elect(&tfull[acc], static_cast<uint16_t>(0x3u << (2 * pp)));
        __syncwarp();
      }
    }
  } else {
    // ===================== epilogue (warps 2..9: two groups) =====================
    // n_sub = 1: group g drains accumulator g (units i = g, g + 2, ...);
    // n_sub = 2: both groups drain every unit, group g its N sub-tile g.
    const int quarter = warp & 3;        // TMEM lanes [32 quarter, 32 quarter + 32)
    const int group = (warp - 2) >> 2;
    constexpr int kOutElt = kTF32 ? 4 : 2;
    constexpr int kPw = 128 / kOutElt;   // columns per 128-byte staging row
    const uint32_t stg = ptx::smem_u32(stg_base) + static_cast<uint32_t>(warp - 2) * kStageOut;
    const uint32_t my_row_s = stg + static_cast<uint32_t>(lane) * 128u;
    const uint32_t my_x = static_cast<uint32_t>(lane & 7);
    const uint32_t tempty0 = ptx::mapa_shared(ptx::smem_u32(tempty), leader_rank);
    const int m = quarter * 32 + lane;   // this thread's row of the CTA's 128
    const int n_c4 = p.bn / 4;           // 16-byte fp32 chunks per partial row (one N sub-tile)
    const int step = p.n_sub == 1 ? 2 : 1;
    int64_t i = p.n_sub == 1 ? group : 0;
    for (int64_t u = pair + i * n_pairs; u < p.n_groups; u += step * n_pairs, i += step) {
      const Unit c = decode_unit(p, u, pp);
      const int acc = p.n_sub == 1 ? group : 0;
      const int sub = p.n_sub == 1 ? 0 : group;  // N sub-tile of this group
      const int64_t use = p.n_sub == 1 ? (i >> 1) : i;
      ptx::mbar_wait(&tfull[acc], static_cast<uint32_t>(use) & 1u);
      ptx::tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                             static_cast<uint32_t>((acc + sub) * p.bn);
      const int64_t r0 = c.mt * kPairM + rank * kBM + quarter * 32;  // first row of this warp
      const int64_t row = r0 + lane;
      const int64_t ncol0 = (static_cast<int64_t>(c.ng) * p.n_sub + sub) * p.bn;  // first output channel
      // this lane's output row O[n, h, w, ncol0 ...] (n-h-w-c: Alg.2 l.17-19 at store time)
      unsigned char* orow = nullptr;
      if (row < p.rows) {
        const int64_t n = static_cast<uint32_t>(row) / static_cast<uint32_t>(p.o_w), w = row - n * p.o_w;  // rows < 2^31
        orow = static_cast<unsigned char*>(p.O) + ((((n * p.o_h + c.h) * p.o_w + w) * p.k_c) + ncol0) * kOutElt;
      }
      const int64_t rem = p.rows - r0;
      const int nvalid = rem <= 0 ? 0 : (rem < 32 ? static_cast<int>(rem) : 32);
      const int64_t cols_left = p.k_c - ncol0;
      bool store = cols_left > 0 && c.valid;
      // split-K slots of this (tile, rank, N sub-tile): chunk-major, 16-byte
      // chunk q of row m at (q * 128 + m) * 16, a warp's store is 512 contiguous bytes
      const int64_t slot_elems = static_cast<int64_t>(n_c4) * kBM;  // float4s per slot
      // (hybrid split: the split tiles are the ones from g_full on -- tile ==
      // unit group index with one pair per cluster -- and only they have slots)
      const float4* part_t = reinterpret_cast<const float4*>(p.part) +
                             (((c.tile - p.g_full) * p.S * 2 + rank) * p.n_sub + sub) * slot_elems;
      const int64_t k_stride = 2 * p.n_sub * slot_elems;  // next range of the same tile
      // output chunks of kPw columns; with split-K, range k owns (reduces and
      // stores) the chunks ci with ci S / n_oc == k and hands the others over
      const int n_oc = (p.bn + kPw - 1) / kPw;  // (bn a multiple of 32: the last chunk may be half)
      if (c.nsplit > 1 && c.valid) {
        float4* mine = const_cast<float4*>(part_t) + c.ks * k_stride;
#pragma unroll 1
        for (int ci = 0; ci < n_oc && !(p.dbg & 2); ++ci) {
          if (ci * c.nsplit / n_oc == c.ks) continue;  // own chunk: stays in TMEM
#pragma unroll
          for (int h16 = 0; h16 < kPw / 16; ++h16) {
            const int c0 = ci * kPw + 16 * h16;
            if (c0 >= p.bn) break;
            uint32_t v[16];
            ptx::tmem_ld_32x32b_x16(taddr + c0, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 4; ++q)
              __stcg(mine + static_cast<int64_t>(c0 / 4 + q) * kBM + m,
                     make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                 __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
          }
        }
        // release the hand-over, then wait until every range of this tile has
        // handed over (the S ranges are co-resident units of the persistent grid:
        // each writes before it waits, and a wait targets the same tile only)
        __threadfence();
        __syncwarp();
        uint32_t* cnt = &p.cnt[(((c.tile * 2 + rank) * 4 + quarter) * p.n_sub) + sub];
        if (lane == 0) atomicAdd(cnt, 1u);
        bool owns = false;  // (S > n_oc: some ranges own no chunk)
        for (int ci = 0; ci < n_oc; ++ci) owns = owns || ci * c.nsplit / n_oc == c.ks;
        store = store && owns;
        if (store) {
          if (lane == 0 && !(p.dbg & 1))
            while (ptx::ld_relaxed_gpu_u32(cnt) < static_cast<uint32_t>(c.nsplit)) __nanosleep(64);
          __syncwarp();
          __threadfence();  // (acquire: the other ranges' partials are read after this)
        }
      }
      if (store) {
#pragma unroll 1
        for (int ci = 0; ci < n_oc && ci * kPw < cols_left; ++ci) {
          if (c.nsplit > 1 && ci * c.nsplit / n_oc != c.ks) continue;
          const int c0 = ci * kPw;
          // split-K, S = 2: the other range's partial, 32 columns (8 loads per
          // thread) in flight ahead of the block being summed (fp32 addition
          // commutes: own + other is the range-order sum)
          const float4* src2 = part_t + (1 - c.ks) * k_stride + static_cast<int64_t>(c0 / 4) * kBM + m;
          float4 x2[8];
          if (c.nsplit == 2 && !(p.dbg & 1)) {
#pragma unroll
            for (int q = 0; q < 8; ++q) x2[q] = __ldcg(src2 + static_cast<int64_t>(q) * kBM);
          }
#pragma unroll 1
          for (int sb = 0; sb < kPw / 32; ++sb) {
            // 32 columns: TMEM (this range) [+ the other ranges' partials, in
            // range order 0, 1, ..., S-1] -> packed -> swizzled staging
            const int cb = c0 + 32 * sb;
            if (cb >= p.bn) break;
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x16(taddr + cb, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
            ptx::tmem_ld_32x32b_x16(taddr + cb + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
            ptx::tmem_ld_wait();
            if (c.nsplit == 2 && !(p.dbg & 1)) {
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 t = x2[q];
                v[4 * q] = __float_as_uint(__uint_as_float(v[4 * q]) + t.x);
                v[4 * q + 1] = __float_as_uint(__uint_as_float(v[4 * q + 1]) + t.y);
                v[4 * q + 2] = __float_as_uint(__uint_as_float(v[4 * q + 2]) + t.z);
                v[4 * q + 3] = __float_as_uint(__uint_as_float(v[4 * q + 3]) + t.w);
              }
              if (sb + 1 < kPw / 32 && cb + 32 < p.bn) {  // the next block's loads, in flight while this one is staged
#pragma unroll
                for (int q = 0; q < 8; ++q) x2[q] = __ldcg(src2 + static_cast<int64_t>(8 * (sb + 1) + q) * kBM);
              }
            } else if (c.nsplit > 2 && !(p.dbg & 1)) {
              // 16 columns at a time (register budget of the 10-warp CTA)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                float a[16];
#pragma unroll 1
                for (int k = 0; k < c.nsplit; ++k) {
                  float x[16];
                  if (k == c.ks) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) x[j] = __uint_as_float(v[16 * h + j]);
                  } else {
                    const float4* src = part_t + k * k_stride + static_cast<int64_t>((cb + 16 * h) / 4) * kBM + m;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                      const float4 t = __ldcg(src + static_cast<int64_t>(q) * kBM);
                      x[4 * q] = t.x;
                      x[4 * q + 1] = t.y;
                      x[4 * q + 2] = t.z;
                      x[4 * q + 3] = t.w;
                    }
                  }
#pragma unroll
                  for (int j = 0; j < 16; ++j) a[j] = k == 0 ? x[j] : a[j] + x[j];
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) v[16 * h + j] = __float_as_uint(a[j]);
              }
            }
            if constexpr (kTF32) {  // 32 fp32 columns = the whole 128-byte row, 8 chunks
#pragma unroll
              for (int ch = 0; ch < 8; ++ch)
                ptx::st_shared_v4(my_row_s + ((static_cast<uint32_t>(ch) ^ my_x) << 4), v[4 * ch], v[4 * ch + 1],
                                  v[4 * ch + 2], v[4 * ch + 3]);
            } else {  // 32 bf16 columns = 64 bytes, chunks 4 sb .. 4 sb + 3
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t ch = static_cast<uint32_t>(4 * sb + q);
                ptx::st_shared_v4(my_row_s + ((ch ^ my_x) << 4),
                                  pack_bf16x2(__uint_as_float(v[8 * q]), __uint_as_float(v[8 * q + 1])),
                                  pack_bf16x2(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3])),
                                  pack_bf16x2(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5])),
                                  pack_bf16x2(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7])));
              }
            }
          }
          __syncwarp();
          // coalesced stores: 8 lanes per 128-byte row segment, 4 rows per instruction
          const int64_t chunks_left = (cols_left - c0) * kOutElt / 16;
          const int nch = chunks_left < 8 ? static_cast<int>(chunks_left) : 8;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int ci2 = it * 32 + lane;
            const int r = ci2 >> 3, ch = ci2 & 7;
            const unsigned long long base = __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(orow), r);
            const uint4 val = ptx::ld_shared_v4(stg + static_cast<uint32_t>(r * 128) +
                                                ((static_cast<uint32_t>(ch) ^ static_cast<uint32_t>(r & 7)) << 4));
            if (r < nvalid && ch < nch)
              *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(base) + c0 * kOutElt + ch * 16) = val;
          }
          __syncwarp();
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(tempty0 + static_cast<uint32_t>(acc) * 8u);
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();  // both CTAs done (no MMA, commit or remote arrive in flight)
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair(tmem_base, 512);
  }
}

// host-side geometry of one call: N sub-tiles per unit, tiles, split count
struct WideGeo {
  int n_sub, n_ng, n_atoms, S, apk;
  int64_t n_mt, tiles;
  int64_t g_full;  // hybrid split: tiles run whole (whole waves) before the split ones
  size_t cnt_words, cnt_bytes, part_bytes;
};

WideGeo wide_geo(const Plan& pl, int split) {
  WideGeo g{};
  // k_c in (256, 512]: both N tiles in one unit (N = 2 bn, the whole TMEM),
  // so A is streamed once for both (48 instead of 64 B per MMA cycle per SM)
  // n_sub = 2 (both N tiles of k_c <= 512 in one unit: A streamed once, but one
  // accumulator set, so the epilogue is not overlapped) measured slower than
  // n_sub = 1 at b1024 (cv6 173 vs 155 us, cv12 129 vs 88 us): opt-in only
  g.n_sub = 1;
  if (const char* e = getenv("MEC_WIDE_NSUB")) g.n_sub = (atoi(e) == 2 && pl.n_tiles_n % 2 == 0) ? 2 : 1;
  g.n_ng = pl.n_tiles_n / g.n_sub;
  g.n_mt = (pl.s.i_n * pl.o_w + kPairM - 1) / kPairM;
  g.tiles = pl.o_h * g.n_mt * g.n_ng;
  g.n_atoms = static_cast<int>(pl.kdim_pad / pl.bk);
  // the pair count is the SM count / 2 here, at plan time and at launch alike,
  // so the workspace sized by the plan always fits the launch
  const int64_t n_pairs = std::max(1, num_sms() / 2);
  g.g_full = 0;
  if (split > 0) {
    g.S = std::min(split, g.n_atoms);
  } else {
    // the split minimising waves x (a range's atoms x n_sub + ~3 atoms of
    // epilogue) + the split's cost: partials written, fenced and counted, and
    // summed by the last range, ~10 + 8 S atom-times (calibrated on B200 at
    // b128: cv11 S = 2 cost 10 us over S = 1 for the same number of atom-waves;
    // cv12, 30 tiles for 74 pairs, gains 36.7 -> 30.5 us with S = 2)
    double best_t = 1e300;
    g.S = 1;
    for (int s = 1; s <= kMaxSplit && s <= std::max(1, g.n_atoms / 4); ++s) {
      const int a = (g.n_atoms + s - 1) / s;
      const int64_t waves = (g.tiles * s + n_pairs - 1) / n_pairs;
      const double t = static_cast<double>(waves) * (a * g.n_sub + 3.0) + (s > 1 ? (10.0 + 8.0 * s) * g.n_sub : 0.0);
      if (t < best_t - 1e-9) {
        best_t = t;
        g.S = s;
      }
    }
    // hybrid: the whole waves of tiles unsplit, the last partial wave's r
    // tiles split into floor(n_pairs / r) ranges (one wave of ranges, each
    // pair at most one): the last wave's time drops from a tile's atoms to a
    // range's, for one exchange (cv12 b128 measured ~3 us ~ 8 atom-times)
    g.g_full = 0;
    const int64_t full = g.tiles / n_pairs * n_pairs, r = g.tiles - full;
    if (full > 0 && r > 0) {
      const int st = static_cast<int>(std::min<int64_t>({kMaxSplit, n_pairs / r, std::max(1, g.n_atoms / 4)}));
      if (st >= 2) {
        const int a = (g.n_atoms + st - 1) / st;
        const double t = static_cast<double>(full / n_pairs) * (g.n_atoms * g.n_sub + 3.0) + (a * g.n_sub + 3.0) +
                         (4.0 + 2.0 * st) * g.n_sub;
        bool use = t < best_t - 1e-9;
        if (const char* e = getenv("MEC_WIDE_HYBRID")) use = atoi(e) != 0;
        if (use) {
          g.S = st;
          g.g_full = full;
        }
      }
    }
    if (const char* e = getenv("MEC_WIDE_SPLIT")) {
      g.S = std::max(1, std::min(g.n_atoms, atoi(e)));
      g.g_full = 0;
    }
  }
  g.apk = (g.n_atoms + g.S - 1) / g.S;
  g.S = (g.n_atoms + g.apk - 1) / g.apk;  // no empty ranges
  g.cnt_words = static_cast<size_t>(g.tiles) * 8 * g.n_sub;
  g.cnt_bytes = (g.cnt_words * sizeof(uint32_t) + 1023) / 1024 * 1024;
  // partial slots for the split tiles only (hybrid: the tail after g_full)
  g.part_bytes = g.S > 1 ? static_cast<size_t>(g.tiles - g.g_full) * g.S * kPairM * g.n_sub * pl.bn * sizeof(float) : 0;
  return g;
}

}  // namespace

bool wide_eligible(const Plan& pl, bool batch_folded, bool fused) {
  // Solution A: the batch-folded rows n o_w + w of Alg.2 l.9's L matrix, 256
  // per pair tile (rows of several images share a tile; the epilogue computes
  // each row's own output address)
  if (fused || !batch_folded) return false;
  if (pl.bn < 64 || pl.bn % 32 != 0) return false;          // N/2 rows of B per CTA, 16-aligned
  if ((pl.s.k_c * pl.elt) % 16 != 0) return false;           // 16-byte output stores
  if (pl.kdim_pad / pl.bk < 2) return false;
  if (pl.s.i_n * pl.o_w >= (1LL << 31)) return false;
  return true;
}

// The weights straight from K as an MN-major B operand (no prepared Kt, so the
// lowering launch does no weight prep): each CTA's N/2 columns must be whole
// 128-byte boxes.  Opt-in (MEC_WIDE_KMN=1): measured on B200 it is correct
// but slower -- the GEMM with MN-major B runs 8-15% longer (cv5 b1024 384 vs
// 332 us, cv12 b1024 103 vs 89 us: twice the B boxes per atom, N-contiguous
// smem reads) while the saved weight prep was only ~2.5 us of the lowering
// launch (its prep CTAs overlap the lowering CTAs).  bf16 only: tf32
// MN-major B in the plain 128-byte swizzle gave wrong products (CUTLASS pairs
// 32-bit MN-major operands with the 128B_BASE32B swizzle).
bool wide_reads_k(const Plan& pl) {
  const char* e = getenv("MEC_WIDE_KMN");
  if (e == nullptr || atoi(e) == 0) return false;
  if (pl.elt != 2) return false;
  const int chunk_n = kTileKBytes / pl.elt;
  return (pl.bn / 2) % chunk_n == 0 && (pl.s.k_c * pl.elt) % 16 == 0;
}

// Tensor-bound: the two-kernel GEMM's arithmetic intensity (SURVEY 8(d):
// (#L + #K + #O) elt bytes) above ~0.8 of the ridge (251 F/B bf16, 126 tf32).
bool wide_preferred(const Plan& pl) {
  if (const char* e = getenv("MEC_WIDE")) return atoi(e) != 0;
  const double flops = 2.0 * pl.s.i_n * pl.o_h * pl.o_w * static_cast<double>(pl.kdim_src) * pl.s.k_c;
  const double bytes = (static_cast<double>(pl.n_L) + static_cast<double>(pl.kdim_src) * pl.s.k_c +
                        static_cast<double>(pl.n_O)) * pl.elt;
  const double ridge = pl.elt == 2 ? 251.0 : 126.0;
  return flops / bytes >= 0.8 * ridge;
}

size_t wide_scratch_bytes(const Plan& pl, int split) {
  const WideGeo g = wide_geo(pl, split);
  return g.cnt_bytes + g.part_bytes;
}

uint32_t wide_zero_words(const Plan& pl) {
  // every split's counters (a forced split_k may differ from the automatic one)
  return static_cast<uint32_t>(wide_geo(pl, 1).cnt_words);
}

cudaError_t launch_wide_gemm(const Plan& pl, const GemmArgs& a, void* scratch, size_t scratch_bytes, int split,
                             cudaStream_t st, int* launches, int* split_used) {
  if (!wide_eligible(pl, a.batch_folded, a.fused) || a.out_hnwc) return cudaErrorNotSupported;
  if (reinterpret_cast<uintptr_t>(a.O) % 16 != 0) return cudaErrorNotSupported;
  const bool tf32 = pl.dt == MEC_DTYPE_TF32;
  const WideGeo g = wide_geo(pl, split);
  WideParams p{};
  p.O = a.O;
  p.o_h = pl.o_h;
  p.o_w = pl.o_w;
  p.i_n = pl.s.i_n;
  p.k_c = pl.s.k_c;
  p.rows = pl.s.i_n * pl.o_w;
  p.n_mt = g.n_mt;
  p.n_sub = g.n_sub;
  p.n_ng = g.n_ng;
  p.bn = pl.bn;
  p.n_var = pl.n_var;
  p.avec = pl.avec;
  p.delta_step = pl.delta_step;
  p.shift = pl.shift;
  p.kc_pad = pl.kc_pad;
  p.bk = pl.bk;
  p.n_atoms = g.n_atoms;
  p.n_tiles = g.tiles;
  p.S = g.S;
  p.apk = g.apk;
  p.dbg = getenv("MEC_WIDE_DBG") ? atoi(getenv("MEC_WIDE_DBG")) : 0;
  p.g_full = g.g_full;
  p.n_units = g.g_full + (g.tiles - g.g_full) * g.S;

  p.a_bytes = static_cast<uint32_t>(kAtomA);
  p.b_half_bytes = static_cast<uint32_t>(pl.bn / 2 * kTileKBytes);
  p.stage_bytes = p.a_bytes + static_cast<uint32_t>(g.n_sub) * p.b_half_bytes;
  const size_t fixed = kSmemAlign + 8 * kStageOut + 64 * 8 + 64;
  p.stages = static_cast<int>(std::min<size_t>(8, (kWideSmemBudget - fixed) / p.stage_bytes));
  if (p.stages < 2) return cudaErrorNotSupported;
  const size_t smem = fixed + static_cast<size_t>(p.stages) * p.stage_bytes;
  if (scratch == nullptr || scratch_bytes < g.cnt_bytes + g.part_bytes) return cudaErrorNotSupported;
  p.cnt = static_cast<uint32_t*>(scratch);
  p.part = reinterpret_cast<float*>(static_cast<unsigned char*>(scratch) + g.cnt_bytes);
  p.b_mn = wide_reads_k(pl) && a.K != nullptr;
  // pairs per cluster sharing one multicast of the weights (MEC_WIDE_MC=2;
  // the prepared K-major weights only).  Opt-in: correct, but measured slower
  // on B200 (cv11 b128 34.8 vs 24.5 us, cv5 b128 61.6 vs 53.1, cv12 b1024
  // 106 vs 89 us) -- the two pairs run in lock step on every stage, which
  // costs more than the halved weight traffic saves (the B300 guide's "TMA
  // multicast ~ unicast at cluster size <= 4")
  p.mc = 1;
  // (one weight copy: the pairs of a cluster may work on different h, whose
  // window alignment would otherwise pick different shifted copies)
  if (const char* e = getenv("MEC_WIDE_MC"))
    p.mc = (atoi(e) == 2 && !p.b_mn && pl.n_var == 1 && g.g_full == 0) ? 2 : 1;
  p.n_hm = pl.o_h * g.n_mt;
  if (p.n_hm * g.n_ng * std::max(1, g.S) >= (1LL << 31)) return cudaErrorNotSupported;  // (32-bit unit decode)
  p.n_groups = p.g_full + (((p.n_hm + p.mc - 1) / p.mc) * g.n_ng - p.g_full) * g.S;
  p.chunk_n = kTileKBytes / pl.elt;
  p.b_chunks = p.b_mn ? (pl.bn / 2) / p.chunk_n : 0;
  p.b_chunk_bytes = static_cast<uint32_t>(kTileKBytes * pl.bk);                 // 128 B x bk K rows
  p.b_kstep16 = static_cast<uint32_t>((32 / pl.elt) * kTileKBytes) >> 4;      // one 32-byte K step of K rows
  p.idesc = ptx::instr_desc(tf32, kPairM, pl.bn, p.b_mn);
  auto kern = tf32 ? (p.mc == 2 ? wide_gemm_kernel<true, 2> : wide_gemm_kernel<true, 1>)
                   : (p.mc == 2 ? wide_gemm_kernel<false, 2> : wide_gemm_kernel<false, 1>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * p.mc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(kWideThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // grid: as many pairs as are co-resident (1 CTA per SM), at most one per unit
  int max_clusters = 0;
  cfg.gridDim = dim3(static_cast<unsigned>(2 * p.mc * std::max(1, num_sms() / (2 * p.mc))));
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
    cudaGetLastError();
    max_clusters = std::max(1, num_sms() / (2 * p.mc));
  }
  // tensor maps: A = L as {i_h k_w i_c, i_n o_w} (pitched rows), B = Kt {kdim_pad, n_var kc_pad}
  CUtensorMap tmA, tmB;
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(pl.l_cols), static_cast<uint64_t>(p.rows)};
    const uint64_t strides[1] = {static_cast<uint64_t>(pl.pitch) * pl.elt};
    const uint32_t box[2] = {static_cast<uint32_t>(pl.bk), static_cast<uint32_t>(kBM)};
    e = encode_tiled(&tmA, tf32, 2, a.L, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  if (p.b_mn) {
    // K_mat = K viewed as (k_h k_w i_c) x k_c row-major (Alg.2 l.7: no copy)
    const uint64_t dims[2] = {static_cast<uint64_t>(pl.s.k_c), static_cast<uint64_t>(pl.kdim_src)};
    const uint64_t strides[1] = {static_cast<uint64_t>(pl.s.k_c) * pl.elt};
    const uint32_t box[2] = {static_cast<uint32_t>(p.chunk_n), static_cast<uint32_t>(pl.bk)};
    e = encode_tiled(&tmB, tf32, 2, a.K, dims, strides, box);
    if (e != cudaSuccess) return e;
  } else {
    const uint64_t dims[2] = {static_cast<uint64_t>(pl.kdim_pad), static_cast<uint64_t>(pl.n_var * pl.kc_pad)};
    const uint64_t strides[1] = {static_cast<uint64_t>(pl.kdim_pad) * pl.elt};
    const uint32_t box[2] = {static_cast<uint32_t>(pl.bk), static_cast<uint32_t>(pl.bn / 2)};
    e = encode_tiled(&tmB, tf32, 2, a.Kt, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  // (the counters were zeroed by the lowering launch: launch_lower's zero_words)
  int64_t clusters = std::min<int64_t>(max_clusters, p.n_groups);
  // hybrid split: the split ranges must form one wave of resident pairs
  // (g_full whole waves before them): else run the plain split model's way
  const bool hybrid_ok = p.g_full > 0 && clusters == std::max(1, num_sms() / 2) && p.g_full % clusters == 0 &&
                         p.n_groups - p.g_full <= clusters;
  if (p.g_full > 0 && !hybrid_ok) {
    p.g_full = 0;
    p.S = 1;
    p.apk = g.n_atoms;
    p.n_units = g.tiles;
    p.n_groups = ((p.n_hm + p.mc - 1) / p.mc) * g.n_ng;
    clusters = std::min<int64_t>(max_clusters, p.n_groups);
  }
  if (p.S > 1 && p.g_full == 0 && clusters < p.n_groups && clusters < 2 * p.S) {
    // the split-K exchange waits on the other ranges of a tile: with fewer
    // resident pairs than 2 S - 1 a pair could wait on a range it would only
    // run itself later (each pair takes units in increasing order, a tile's
    // ranges are S consecutive units) -- run unsplit
    p.S = 1;
    p.apk = g.n_atoms;
    p.n_units = g.tiles;
    p.n_groups = ((p.n_hm + p.mc - 1) / p.mc) * g.n_ng;
    clusters = std::min<int64_t>(max_clusters, p.n_groups);
  }
  cfg.gridDim = dim3(static_cast<unsigned>(2 * p.mc * clusters));
  cfg.numAttrs = getenv("MEC_NO_PDL") ? 1 : 2;
  e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, p);
  if (e != cudaSuccess) return e;
  if (launches) ++*launches;
  if (split_used) *split_used = p.S;
  return cudaGetLastError();
}

}  // namespace mec
