// pair_sweep.cu -- MEC's window GEMMs as an atom-major sweep along h on CTA
// pairs (tcgen05 cta_group::2), for windows larger than the TMEM ring
// (sm_100a).
//
// Paper: output row h is O[:, h] = L[:, h s_h k_w i_c : + k_h k_w i_c] x K
// (Sec. 3.2; Alg.2 l.10-12 Solution A, l.23-25 Solution B).
// Consecutive windows overlap by (k_h - s_h) k_w i_c columns, so a stream of
// L's columns feeds k_h / s_h output rows at once.  The h-sweep kernel
// (sweep_gemm.cu) keeps a whole window in a TMEM ring and issues row by row;
// a window wider than that ring (VGG conv1_2 in tf32: 18 atoms of 128 bytes;
// AlexNet-size kernels) cannot use it, and the one-window kernel re-reads
// every window from L2 k_h / s_h times (L2 -> SM bandwidth is
// about HBM bandwidth, so the GEMM ran at ~3 #L of traffic).
//
// Here every L column is read ONCE per work item and consumed atom-major:
//   * work item = (pair of 128-row CTA tiles of L, chunk of H output rows);
//     its stream is the columns [h0 shift, (h0 + H - 1) shift + kdim) of the
//     tiles' rows (shift a whole number of 128-byte atoms: the windows start
//     on atom boundaries, so no shifted weight copy is needed);
//   * when stream atom j has landed (both CTAs' 128 rows, TMA, one expect_tx
//     on the leader's barrier), the leader issues for every open row r (the
//     rows whose window [r sa, r sa + na) holds j) the 4 MMAs of the atom into
//     r's accumulator, with B = the resident weight atom j - r sa: M = 256
//     (cta_group::2; each CTA's 128 rows of A), N = k_c (each CTA holds k_c/2
//     rows of the weights, resident for the whole kernel);
//   * accumulators rotate through TMEM (n_acc of them, >= open rows + 1); a
//     row's accumulator is committed to the epilogue at its last atom;
//   * 8 epilogue warps (two groups, alternate rows) drain row by row:
//     tcgen05.ld -> bf16 / fp32 -> swizzled smem -> coalesced 16-byte stores
//     of O[n, h, w, :] (n-h-w-c: Solution A's permutation, Alg.2 l.17-19, at
//     store time) or O_hnwc[h, n, w, :].
// Per row the arithmetic is the window's K atoms in order, 4 MMAs each (the
// same K steps as the one-window kernel).
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
// Debug-only cycle accounting (tools/trace_pair_sweep.py, -DMEC_TRACE build):
// per CTA [0] MMA warp cycles waiting for a free accumulator, [1] waiting for
// landed atoms, [2] MMA warp total, [3] producer cycles waiting for a free
// stage, [4] producer total, [5] atoms issued, [6] rows, [7] SM id
__device__ unsigned long long* g_ps_trace = nullptr;
extern "C" int mec_pair_sweep_trace_enable(void** dev_buf_out, size_t* bytes_out) {
  const size_t bytes = static_cast<size_t>(512) * 8 * 8;
  void* buf = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
  cudaMemset(buf, 0, bytes);
  if (cudaMemcpyToSymbol(g_ps_trace, &buf, sizeof(buf)) != cudaSuccess) return 2;
  *dev_buf_out = buf;
  *bytes_out = bytes;
  return 0;
}
#define PS_CLK(v) const long long v = clock64()
#define PS_ADD(acc, t0) acc += clock64() - (t0)
#endif

namespace mec {
namespace {

constexpr int kPsThreads = 64 + 2 * 128;
constexpr uint32_t kPsStageOut = 32 * 128;        // epilogue staging per warp
constexpr size_t kPsSmemBudget = 227 * 1024;
constexpr size_t kPsMaxResident = 112 * 1024;     // per CTA: k_c/2 weight rows x kdim (else streamed)

struct PsParams {
  void* O;
  int64_t o_h, o_w, i_n, k_c;
  bool out_hnwc;
  int ipt, slot;         // image slots per CTA tile (ipt = 1: a CTA tile is 128 rows of one image)
  int64_t mt_per_img;    // ipt = 1: CTA tiles per image
  int64_t n_ctile;       // CTA tiles
  int64_t n_pt;          // pair tiles = ceil(n_ctile / 2)
  int H;                 // output rows per chunk (the last chunk may be shorter)
  int64_t n_hc, n_items;
  // balanced split (bal_P > 0): pair c owns rows [c R / P, (c + 1) R / P) of
  // the flattened (pair tile, h) sequence (R = n_pt o_h), cut at pair-tile
  // boundaries into at most bal_J items; item it = c + j P is piece j of pair c
  int64_t bal_R;
  int bal_P, bal_J;
  int64_t shift;         // elements
  int bk, sa, na;        // atom width (elements), shift atoms, window atoms (kdim_pad / bk)
  int bn;                // MMA N (k_c rounded up to 16)
  int n_acc;             // TMEM accumulators (bn columns each)
  int stages;
  uint32_t a_bytes;      // this CTA's A bytes per atom (TMA boxes)
  uint32_t b_half_bytes; // bn/2 rows x 128 bytes: one weight atom per CTA
  // weights resident (b_stream = false), or streamed with A: stage s holds
  // the A atom and, for each open row, that row's weight atom (b_open slots)
  bool b_stream;
  int b_open;
  int aps;               // stream atoms per pipeline stage (one full/empty handshake and commit each)
  uint32_t slot_bytes;   // one atom of a stage: A (16 KB) [+ b_open x b_half_bytes]
  uint32_t stage_bytes;  // aps x slot_bytes
  uint32_t idesc;
  bool a_evict_first;    // (experiments: MEC_PS_EVICT_FIRST=1) L2 evict-first hint on the L stream
  // streamed weights in ONE 3-D TMA box per atom (tmB3: {kdim_pad, kc_pad,
  // b_open} with the third stride sa atoms): slab z = the weight atom of row
  // r_hi - z (atom j - r_hi sa + z sa); slabs of rows that are not open (item
  // start / end) are loaded and not read.  One issue instead of one per open
  // row: the producer was ~87% busy issuing 5 boxes per cv4 atom
  bool b3;
};

// CTA tile c -> the image and first row (w) of each of its rows' slots
struct CTile {
  int64_t n0;   // first image
  int64_t w0;   // first w (ipt = 1)
};

__device__ __forceinline__ CTile ctile(const PsParams& p, int64_t c) {
  CTile t;
  if (p.ipt == 1) {
    t.n0 = c / p.mt_per_img;
    t.w0 = (c - t.n0 * p.mt_per_img) * kBM;
  } else {
    t.n0 = c * p.ipt;
    t.w0 = 0;
  }
  return t;
}

// work item it -> pair tile pt, first output row h0 and row count (0: an
// empty piece of a balanced split)
__device__ __forceinline__ void ps_item(const PsParams& p, int64_t it, int64_t* pt, int64_t* h0, int* rows) {
  if (p.bal_P > 0) {
    const int64_t c = it % p.bal_P, j = it / p.bal_P;
    const int64_t s = c * p.bal_R / p.bal_P, e = (c + 1) * p.bal_R / p.bal_P;
    const int64_t tile0 = s / p.o_h;
    const int64_t start = j == 0 ? s : (tile0 + j) * p.o_h;
    const int64_t end = min(e, (tile0 + j + 1) * p.o_h);
    if (start >= end) {
      *pt = tile0;
      *h0 = 0;
      *rows = 0;
      return;
    }
    *pt = start / p.o_h;
    *h0 = start - *pt * p.o_h;
    *rows = static_cast<int>(end - start);
    return;
  }
  const int64_t q = it / p.n_hc, hc = it - q * p.n_hc;
  *pt = q;
  *h0 = hc * p.H;
  *rows = static_cast<int>(p.o_h - *h0 < p.H ? p.o_h - *h0 : p.H);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <bool kTF32, int kAps>
__global__ void __launch_bounds__(kPsThreads, 1)
    pair_sweep_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmB3, const PsParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + kSmemAlign - 1) & ~uintptr_t(kSmemAlign - 1));
  const int S = p.stages;
  unsigned char* smemB = smem + static_cast<size_t>(S) * p.stage_bytes;  // resident weights (if any)
  unsigned char* stg_base = smemB + (p.b_stream ? 0 : static_cast<size_t>(p.na) * p.b_half_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg_base + 8 * kPsStageOut);
  uint64_t* full = bars;                  // [S] leader
  uint64_t* empty = bars + S;             // [S] each CTA
  uint64_t* tfull = bars + 2 * S;         // [8] each CTA
  uint64_t* tempty = bars + 2 * S + 8;    // [8] leader
  uint64_t* bfull = bars + 2 * S + 16;    // leader: both CTAs' weights landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 17);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t pair = ptx::cluster_id_x();
  const int64_t n_pairs = ptx::nclusters_x();

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    if (p.b3) ptx::tma_prefetch_desc(&tmB3);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 8; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 8);  // one epilogue group: 4 warps x 2 CTAs
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();      // the allocator's write of tmem_slot before any read (a CTA barrier racecheck models)
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      // L columns are streamed once per item; adjacent chunks of the same tile
      // (run at the same time by neighbouring pairs) share na - sa atoms in L2
      const uint64_t hintA = p.a_evict_first ? ptx::policy_evict_first() : ptx::policy_evict_normal();
      const uint64_t hintB = ptx::policy_evict_last();
      ptx::griddep_wait();  // L and Kt come from the preceding (lowering) kernel
      const uint32_t full0 = ptx::mapa_shared(ptx::smem_u32(full), 0);
      const uint32_t bfull0 = ptx::mapa_shared(ptx::smem_u32(bfull), 0);
      if (pair < p.n_items && !p.b_stream) {
        // this CTA's half of the weights (k_c/2 rows of every window atom), resident
        if (leader) ptx::mbar_arrive_expect_tx(bfull, 2u * static_cast<uint32_t>(p.na) * p.b_half_bytes);
        for (int a = 0; a < p.na; ++a)
          ptx::tma_load_2d_pair(smemB + static_cast<size_t>(a) * p.b_half_bytes, &tmB, bfull0, a * p.bk,
                                static_cast<int32_t>(rank * (p.bn / 2)), hintB);
      }
      int stage = 0;
      uint32_t phase = 0;
#ifdef MEC_TRACE
      long long c_pwait = 0, n_atoms = 0;
      const long long c_p0 = clock64();
#endif
      for (int64_t it = pair; it < p.n_items; it += n_pairs) {
        int64_t pt, h0;
        int rows;
        ps_item(p, it, &pt, &h0, &rows);
        if (rows == 0) continue;
        const int n_stream = (rows - 1) * p.sa + p.na;
        const CTile t = ctile(p, 2 * pt + rank);
        const int32_t x0 = static_cast<int32_t>(h0 * p.shift);
        int k = 0;  // atom slot within the current stage
        // open rows r_lo..r_hi of atom j kept incrementally: no divisions on
        // the producer's per-atom path, which issues 1 + open TMA boxes per
        // atom (cv4 b128 GEMM 958 -> 757 us with the four divisions gone)
        int r_lo = 0, r_hi = -1, next_start = 0, lo_end = p.na - 1;
        for (int j = 0; j < n_stream; ++j) {
          // streamed weights: the open rows r_lo..r_hi of this atom each need weight atom j - r sa
          if (j == next_start) {
            if (r_hi + 1 < rows) ++r_hi;
            next_start += p.sa;
          }
          const uint32_t fb = full0 + static_cast<uint32_t>(stage) * 8u;
          if (k == 0) {  // a new stage: its bytes (up to aps atoms), one expect_tx
            uint32_t bytes = 0;
            if (kAps == 1) {
              bytes = p.a_bytes + (p.b_stream ? static_cast<uint32_t>(p.b3 ? p.b_open : r_hi - r_lo + 1) * p.b_half_bytes
                                              : 0u);
            } else {
              const int na_s = min(kAps, n_stream - j);
              for (int kk = 0; kk < na_s; ++kk) {
                const int jj = j + kk;
                const int hi = min(rows - 1, jj / p.sa);
                const int lo = jj >= p.na ? (jj - p.na) / p.sa + 1 : 0;
                bytes += p.a_bytes + (p.b_stream ? static_cast<uint32_t>(hi - lo + 1) * p.b_half_bytes : 0u);
              }
            }
#ifdef MEC_TRACE
            PS_CLK(tw0);
#endif
            ptx::mbar_wait(&empty[stage], phase ^ 1);
#ifdef MEC_TRACE
            PS_ADD(c_pwait, tw0);
#endif
            if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2u * bytes);
          }
          unsigned char* dA = smem + static_cast<size_t>(stage) * p.stage_bytes + static_cast<size_t>(k) * p.slot_bytes;
          if (p.b3) {
            ptx::tma_load_3d_pair(dA + kBM * kTileKBytes, &tmB3, fb, (j - r_hi * p.sa) * p.bk,
                                  static_cast<int32_t>(rank * (p.bn / 2)), 0, hintB);
          } else if (p.b_stream) {
            for (int r = r_lo; r <= r_hi; ++r)
              ptx::tma_load_2d_pair(dA + kBM * kTileKBytes + (r - r_lo) * p.b_half_bytes, &tmB, fb,
                                    (j - r * p.sa) * p.bk, static_cast<int32_t>(rank * (p.bn / 2)), hintB);
          }
          const int32_t x = x0 + j * p.bk;
          if (p.ipt == 1) {
            ptx::tma_load_3d_pair(dA, &tmA, fb, x, static_cast<int32_t>(t.w0), static_cast<int32_t>(t.n0), hintA);
          } else {
            // one box of ipt images x slot rows (images >= i_n, rows >= o_w: zero fill)
            ptx::tma_load_3d_pair(dA, &tmA, fb, x, 0, static_cast<int32_t>(t.n0), hintA);
          }
#ifdef MEC_TRACE
          ++n_atoms;
#endif
          if (j == lo_end) {  // row r_lo's window ends with this atom
            ++r_lo;
            lo_end += p.sa;
          }
          if (++k == kAps || j == n_stream - 1) {
            k = 0;
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
#ifdef MEC_TRACE
      if (g_ps_trace != nullptr && blockIdx.x < 512) {
        unsigned long long* e = g_ps_trace + static_cast<size_t>(blockIdx.x) * 8;
        e[3] = static_cast<unsigned long long>(c_pwait);
        e[4] = static_cast<unsigned long long>(clock64() - c_p0);
        e[5] = static_cast<unsigned long long>(n_atoms);
      }
#endif
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (pair leader) =====================
    if (leader && pair < p.n_items) {
      const uint64_t adesc0 = ptx::smem_desc_sw128(ptx::smem_u32(smem));
      const uint64_t bdesc0 = ptx::smem_desc_sw128(ptx::smem_u32(smemB));
      const uint32_t a_stage16 = p.stage_bytes >> 4, b16 = p.b_half_bytes >> 4;
      const uint32_t a_to_b16 = (kBM * kTileKBytes) >> 4, slot16 = p.slot_bytes >> 4;
      if (!p.b_stream) ptx::mbar_wait(bfull, 0);
      // Division-free bookkeeping (the MMA warp's scalar code was the limit:
      // 80-90% of its time issuing at ~2x the MMA time per atom, trace build):
      // the open rows r_lo..r_hi, the atom at which the next row starts and the
      // one after which the oldest completes, and the accumulators of the
      // oldest and the next row (rows complete in order; all rows of an item
      // complete before the next item's first row starts)
      int stage = 0;
      uint32_t phase = 0;
      const int sa = p.sa, na = p.na;
      const uint32_t n_acc = static_cast<uint32_t>(p.n_acc), bn = static_cast<uint32_t>(p.bn);
      uint32_t acc_lo = 0, acc_next = 0, tph_next = 0;
#ifdef MEC_TRACE
      long long c_tempty = 0, c_full = 0;
      uint32_t rows_total = 0;
      const long long c_m0 = clock64();
#endif
      for (int64_t it = pair; it < p.n_items; it += n_pairs) {
        int64_t pt_, h0_;
        int rows;
        ps_item(p, it, &pt_, &h0_, &rows);
        if (rows == 0) continue;
        const int n_stream = (rows - 1) * sa + na;
#ifdef MEC_TRACE
        rows_total += static_cast<uint32_t>(rows);
#endif
        int k = 0;  // atom slot within the current stage
        int r_lo = 0, r_hi = -1;
        int next_start = 0;  // atom at which row r_hi + 1 starts
        int lo_start = 0;    // atom at which row r_lo started (its window atom = j - lo_start)
        for (int j = 0; j < n_stream; ++j) {
          if (j == next_start) {
            if (r_hi + 1 < rows) {
              // row r_hi + 1 starts here: its accumulator must be drained
              ++r_hi;
#ifdef MEC_TRACE
              PS_CLK(t0);
#endif
              ptx::mbar_wait(&tempty[acc_next], tph_next ^ 1u);
#ifdef MEC_TRACE
              PS_ADD(c_tempty, t0);
#endif
              if (++acc_next == n_acc) {
                acc_next = 0;
                tph_next ^= 1u;
              }
            }
            next_start += sa;
          }
#ifdef MEC_TRACE
          PS_CLK(t1);
#endif
          if (k == 0) ptx::mbar_wait(&full[stage], phase);
#ifdef MEC_TRACE
          PS_ADD(c_full, t1);
#endif
          ptx::tc_fence_after();
          const uint64_t ad = adesc0 + static_cast<uint32_t>(stage) * a_stage16 + static_cast<uint32_t>(k) * slot16;
          // rows r_lo..r_hi: window atom a = j - r sa, accumulator acc_lo + (r - r_lo);
          // weights: the atom slot's weight part r - r_lo (streamed) or resident atom a
          int a = j - lo_start;
          uint32_t acc = acc_lo;
          // (3-D weight box: row r's slab is z = r_hi - r, so the rows walk it backwards)
          uint64_t bd = p.b3 ? ad + a_to_b16 + static_cast<uint32_t>(r_hi - r_lo) * b16
                             : (p.b_stream ? ad + a_to_b16 : bdesc0 + static_cast<uint32_t>(a) * b16);
          const int64_t bstep = p.b3 ? -static_cast<int64_t>(b16)
                                     : (p.b_stream ? static_cast<int64_t>(b16) : -static_cast<int64_t>(sa) * b16);
          for (int r = r_lo; r <= r_hi; ++r) {
            ptx::mma_ss_atom_pair_elect<kTF32>(tmem_base + acc * bn, ad, bd, p.idesc, a != 0 ? 1u : 0u);
            if (++acc == n_acc) acc = 0;
            a -= sa;
            bd += static_cast<uint64_t>(bstep);
          }
          const bool stage_end = ++k == kAps || j == n_stream - 1;
          if (stage_end) ptx::mma_commit_pair_elect(&empty[stage], 0x3);  // one release per stage of aps atoms
          if (j - lo_start == na - 1) {  // the oldest open row is complete
            ptx::mma_commit_pair_elect(&tfull[acc_lo], 0x3);
            ++r_lo;
            lo_start += sa;
            if (++acc_lo == n_acc) acc_lo = 0;
          }
          __syncwarp();
          if (stage_end) {
            k = 0;
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
#ifdef MEC_TRACE
      if (lane == 0 && g_ps_trace != nullptr && blockIdx.x < 512) {
        unsigned long long* e = g_ps_trace + static_cast<size_t>(blockIdx.x) * 8;
        e[0] = static_cast<unsigned long long>(c_tempty);
        e[1] = static_cast<unsigned long long>(c_full);
        e[2] = static_cast<unsigned long long>(clock64() - c_m0);
        e[6] = rows_total;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        e[7] = smid;
      }
#endif
    }
  } else {
    // ===================== epilogue (warps 2..9: two groups, alternate rows) =====================
    const int quarter = warp & 3;
    const int group = (warp - 2) >> 2;
    constexpr int kOutElt = kTF32 ? 4 : 2;
    constexpr int kPw = 128 / kOutElt;
    const uint32_t stg = ptx::smem_u32(stg_base) + static_cast<uint32_t>(warp - 2) * kPsStageOut;
    const uint32_t my_row_s = stg + static_cast<uint32_t>(lane) * 128u;
    const uint32_t my_x = static_cast<uint32_t>(lane & 7);
    const uint32_t tempty0 = ptx::mapa_shared(ptx::smem_u32(tempty), 0);
    const int m = quarter * 32 + lane;
    const int64_t cols_left = p.k_c;
    uint32_t row_seq = 0;
    for (int64_t it = pair; it < p.n_items; it += n_pairs) {
      int64_t pt, h0;
      int rows;
      ps_item(p, it, &pt, &h0, &rows);
      if (rows == 0) continue;
      const CTile t = ctile(p, 2 * pt + rank);
      // this thread's row of the tile: image n, column w
      int64_t n, w;
      bool valid;
      if (p.ipt == 1) {
        n = t.n0;
        w = t.w0 + m;
        valid = w < p.o_w && n < p.i_n;
      } else {
        const int s = m / p.slot;
        n = t.n0 + s;
        w = m - s * p.slot;
        valid = s < p.ipt && w < p.o_w && n < p.i_n;
      }
      for (int r = 0; r < rows; ++r) {
        const uint32_t q = row_seq + static_cast<uint32_t>(r);
        if (static_cast<int>(q & 1u) != group) continue;
        const int acc = static_cast<int>(q % p.n_acc);
        ptx::mbar_wait(&tfull[acc], (q / p.n_acc) & 1u);
        ptx::tc_fence_after();
        const int64_t h = h0 + r;
        unsigned char* orow = nullptr;
        if (valid) {
          const int64_t out_row = p.out_hnwc ? (h * p.i_n + n) * p.o_w + w : (n * p.o_h + h) * p.o_w + w;
          orow = static_cast<unsigned char*>(p.O) + out_row * p.k_c * kOutElt;
        }
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                               static_cast<uint32_t>(acc * p.bn);
        if (!kTF32 && p.bn == 128 && cols_left >= 128) {
          // bf16, N = 128 (cv8): the whole row out of TMEM first, packed to
          // bf16 (64 registers), then the accumulator is released BEFORE the
          // stores -- with 4 accumulators for 3 open rows the MMA warp waited
          // a third of its time for a drained one (trace build)
          uint32_t pk[64];
#pragma unroll
          for (int cb = 0; cb < 128; cb += 32) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x16(taddr + cb, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
            ptx::tmem_ld_32x32b_x16(taddr + cb + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
            ptx::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[cb / 2 + e] = pack_bf16x2(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(tempty0 + static_cast<uint32_t>(acc) * 8u);
#pragma unroll
          for (int c0 = 0; c0 < 128; c0 += kPw) {
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const uint32_t* w4 = &pk[c0 / 2 + 4 * ch];
              ptx::st_shared_v4(my_row_s + ((static_cast<uint32_t>(ch) ^ my_x) << 4), w4[0], w4[1], w4[2], w4[3]);
            }
            __syncwarp();
#pragma unroll
            for (int i2 = 0; i2 < 8; ++i2) {
              const int ci = i2 * 32 + lane;
              const int rr = ci >> 3, ch = ci & 7;
              const unsigned long long base = __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(orow), rr);
              const uint4 val = ptx::ld_shared_v4(stg + static_cast<uint32_t>(rr * 128) +
                                                  ((static_cast<uint32_t>(ch) ^ static_cast<uint32_t>(rr & 7)) << 4));
              if (base != 0ull)
                *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(base) + c0 * kOutElt + ch * 16) = val;
            }
            __syncwarp();
          }
          continue;
        }
        for (int c0 = 0; c0 < p.bn && c0 < cols_left; c0 += kPw) {
#pragma unroll
          for (int sb = 0; sb < kPw / 32; ++sb) {
            const int cb = c0 + 32 * sb;
            if (cb >= p.bn) break;  // (bf16 with bn = 16 or 48 ...: a half-filled staging row)
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x16(taddr + cb, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
            if (cb + 16 < p.bn) ptx::tmem_ld_32x32b_x16(taddr + cb + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
            ptx::tmem_ld_wait();
            if constexpr (kTF32) {
#pragma unroll
              for (int ch = 0; ch < 8; ++ch)
                ptx::st_shared_v4(my_row_s + ((static_cast<uint32_t>(ch) ^ my_x) << 4), v[4 * ch], v[4 * ch + 1],
                                  v[4 * ch + 2], v[4 * ch + 3]);
            } else {
#pragma unroll
              for (int qq = 0; qq < 4; ++qq) {
                const uint32_t ch = static_cast<uint32_t>(4 * sb + qq);
                ptx::st_shared_v4(my_row_s + ((ch ^ my_x) << 4),
                                  pack_bf16x2(__uint_as_float(v[8 * qq]), __uint_as_float(v[8 * qq + 1])),
                                  pack_bf16x2(__uint_as_float(v[8 * qq + 2]), __uint_as_float(v[8 * qq + 3])),
                                  pack_bf16x2(__uint_as_float(v[8 * qq + 4]), __uint_as_float(v[8 * qq + 5])),
                                  pack_bf16x2(__uint_as_float(v[8 * qq + 6]), __uint_as_float(v[8 * qq + 7])));
              }
            }
          }
          __syncwarp();
          const int64_t chunks_left = (cols_left - c0) * kOutElt / 16;
          const int nch = chunks_left < 8 ? static_cast<int>(chunks_left) : 8;
#pragma unroll
          for (int i2 = 0; i2 < 8; ++i2) {
            const int ci = i2 * 32 + lane;
            const int rr = ci >> 3, ch = ci & 7;
            const unsigned long long base = __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(orow), rr);
            const uint4 val = ptx::ld_shared_v4(stg + static_cast<uint32_t>(rr * 128) +
                                                ((static_cast<uint32_t>(ch) ^ static_cast<uint32_t>(rr & 7)) << 4));
            if (base != 0ull && ch < nch)
              *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(base) + c0 * kOutElt + ch * 16) = val;
          }
          __syncwarp();
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(tempty0 + static_cast<uint32_t>(acc) * 8u);
      }
      row_seq += static_cast<uint32_t>(rows);
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair(tmem_base, 512);
  }
}

struct PsGeo {
  int ipt, slot;
  int64_t mt_per_img, n_ctile, n_pt;
  int sa, na, n_acc, stages;
  uint32_t a_bytes, b_half_bytes, stage_bytes, slot_bytes;
  int aps;
  bool b_stream;
  int b_open;
  size_t smem;
};

bool ps_geo(const Plan& pl, bool batch_folded, PsGeo* g) {
  if (pl.n_tiles_n != 1 || pl.n_var != 1 || pl.o_h < 2) return false;
  if (pl.shift % pl.bk != 0 || pl.shift >= pl.kdim) return false;  // windows on atom boundaries, overlapping
  if (pl.o_w < 32 && batch_folded) return false;                     // flat Solution A rows: the other kernels
  if (pl.l_cols > (1LL << 30) || pl.o_h * pl.shift > (1LL << 30)) return false;
  if ((pl.s.k_c * pl.elt) % 16 != 0 || pl.bn % 16 != 0) return false;
  g->sa = static_cast<int>(pl.shift / pl.bk);
  g->na = static_cast<int>(pl.kdim_pad / pl.bk);
  g->ipt = 1;
  g->slot = kBM;
  if (batch_folded && pl.o_w <= 128) {
    const int slot = static_cast<int>((pl.o_w + 31) / 32 * 32);
    g->ipt = std::max(1, kBM / slot);
    if (g->ipt > 1) g->slot = slot;
  }
  g->mt_per_img = g->ipt == 1 ? (pl.o_w + kBM - 1) / kBM : 1;
  g->n_ctile = g->ipt == 1 ? pl.s.i_n * g->mt_per_img : (pl.s.i_n + g->ipt - 1) / g->ipt;
  g->n_pt = (g->n_ctile + 1) / 2;
  const int open = (g->na + g->sa - 1) / g->sa;  // rows a stream atom can feed
  g->n_acc = std::min(8, 512 / pl.bn);
  if (g->n_acc < open + 1) return false;
  g->b_half_bytes = static_cast<uint32_t>(pl.bn / 2 * kTileKBytes);
  size_t b_res = static_cast<size_t>(g->na) * g->b_half_bytes;
  // weights that do not fit resident (cv4: 49 atoms) are streamed with A: the
  // open rows' weight atoms ride in the stage (<= `open` x k_c/2 rows)
  g->b_stream = b_res > kPsMaxResident || (getenv("MEC_PS_BSTREAM") && atoi(getenv("MEC_PS_BSTREAM")) != 0);
  g->b_open = open;
  if (g->b_stream) b_res = 0;
  g->a_bytes = static_cast<uint32_t>(g->ipt == 1 ? kBM * kTileKBytes : g->ipt * g->slot * kTileKBytes);
  g->slot_bytes = static_cast<uint32_t>(kBM * kTileKBytes + (g->b_stream ? open * g->b_half_bytes : 0));
  const size_t fixed = kSmemAlign + b_res + 8 * kPsStageOut + 32 * 8 + 64;
  // atoms per stage: 1 (one full/empty handshake and commit per atom).  2-3
  // atoms per stage (MEC_PS_APS, experiments) measured slower on B200: C2 tf32
  // 701 -> 767 / 795 us, cv4 b128 936 -> 1258 / 1233 us (fewer stages in
  // flight; the per-atom commits are not the bottleneck here)
  g->aps = 1;
  if (const char* e = getenv("MEC_PS_APS")) g->aps = std::max(1, std::min(3, atoi(e)));
  g->stage_bytes = static_cast<uint32_t>(g->aps) * g->slot_bytes;
  const size_t stage = g->stage_bytes;
  if (fixed + 2 * stage > kPsSmemBudget) return false;
  g->stages = static_cast<int>(std::min<size_t>(12, (kPsSmemBudget - fixed) / stage));
  g->smem = fixed + g->stages * stage;
  return true;
}

}  // namespace

bool pair_sweep_eligible(const Plan& pl, bool batch_folded, bool fused) {
  PsGeo g;
  return !fused && ps_geo(pl, batch_folded, &g);
}

cudaError_t launch_pair_sweep(const Plan& pl, const GemmArgs& a, cudaStream_t st, int* launches) {
  PsGeo g;
  if (a.fused || !ps_geo(pl, a.batch_folded, &g)) return cudaErrorNotSupported;
  if (reinterpret_cast<uintptr_t>(a.O) % 16 != 0) return cudaErrorNotSupported;
  const bool tf32 = pl.dt == MEC_DTYPE_TF32;
  PsParams p{};
  p.O = a.O;
  p.o_h = pl.o_h;
  p.o_w = pl.o_w;
  p.i_n = pl.s.i_n;
  p.k_c = pl.s.k_c;
  p.out_hnwc = a.out_hnwc;
  p.ipt = g.ipt;
  p.slot = g.slot;
  p.mt_per_img = g.mt_per_img;
  p.n_ctile = g.n_ctile;
  p.n_pt = g.n_pt;
  p.shift = pl.shift;
  p.bk = pl.bk;
  p.sa = g.sa;
  p.na = g.na;
  p.bn = pl.bn;
  p.n_acc = g.n_acc;
  p.stages = g.stages;
  p.a_bytes = g.a_bytes;
  p.b_half_bytes = g.b_half_bytes;
  p.b_stream = g.b_stream;
  p.b_open = g.b_open;
  p.stage_bytes = g.stage_bytes;
  p.slot_bytes = g.slot_bytes;
  p.aps = g.aps;
  p.a_evict_first = getenv("MEC_PS_EVICT_FIRST") && atoi(getenv("MEC_PS_EVICT_FIRST")) != 0;
  p.idesc = ptx::instr_desc(tf32, 2 * kBM, pl.bn);
  // atoms per stage as a template parameter: the 1-atom instance keeps the
  // per-atom loop free of stage bookkeeping (a runtime aps cost ~30% there)
  auto kern = tf32 ? (g.aps == 1 ? pair_sweep_kernel<true, 1> : g.aps == 2 ? pair_sweep_kernel<true, 2>
                                                                           : pair_sweep_kernel<true, 3>)
                   : (g.aps == 1 ? pair_sweep_kernel<false, 1> : g.aps == 2 ? pair_sweep_kernel<false, 2>
                                                                            : pair_sweep_kernel<false, 3>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(g.smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(kPsThreads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;
  cfg.gridDim = dim3(static_cast<unsigned>(2 * std::max(1, num_sms() / 2)));
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
    cudaGetLastError();
    max_clusters = std::max(1, num_sms() / 2);
  }
  // output-row chunks: the H minimising waves x streamed atoms per item
  int64_t best_hc = 1;
  double best_t = 1e300;
  for (int64_t hc = 1; hc <= std::min<int64_t>(pl.o_h, 64); ++hc) {
    const int64_t H = (pl.o_h + hc - 1) / hc;
    const int64_t items = g.n_pt * ((pl.o_h + H - 1) / H);
    const int64_t waves = (items + max_clusters - 1) / max_clusters;
    const double t = static_cast<double>(waves) * ((H - 1) * g.sa + g.na + 4);
    if (t < best_t - 1e-9) {
      best_t = t;
      best_hc = hc;
    }
  }
  // balanced split: each pair the same number of (pair tile, h) rows, cut at
  // pair-tile boundaries (<= 2 pieces when a pair's share is at most one
  // tile's rows), where the wave model prefers it to the chunks -- no idle
  // pairs (cv4 / cv8 at b128: 64 pair tiles of one chunk for 74 pairs) and no
  // partial last wave (C2 tf32); cost = its pieces' streams
  bool balanced = false;
  const int64_t R = g.n_pt * pl.o_h, P = max_clusters;
  if (R >= P) {
    double worst = 0.0;
    for (int64_t c = 0; c < P; ++c) {
      const int64_t s0 = c * R / P, e0 = (c + 1) * R / P;
      double t = 0.0;
      for (int64_t pos = s0; pos < e0;) {
        const int64_t end = std::min(e0, (pos / pl.o_h + 1) * pl.o_h);
        t += static_cast<double>((end - pos - 1) * g.sa + g.na + 4);
        pos = end;
      }
      worst = std::max(worst, t);
    }
    balanced = worst < best_t * 0.999;
  }
  if (const char* e3 = getenv("MEC_PS_BALANCED")) balanced = atoi(e3) != 0 && R >= P;
  if (const char* e2 = getenv("MEC_PS_CHUNKS")) {
    best_hc = std::max<int64_t>(1, std::min<int64_t>(pl.o_h, atoi(e2)));
    balanced = false;
  }
  p.H = static_cast<int>((pl.o_h + best_hc - 1) / best_hc);
  p.n_hc = (pl.o_h + p.H - 1) / p.H;
  p.n_items = g.n_pt * p.n_hc;
  if (balanced) {
    p.bal_R = R;
    p.bal_P = static_cast<int>(P);
    p.bal_J = static_cast<int>(((R + P - 1) / P + pl.o_h - 1) / pl.o_h + 1);
    p.n_items = P * p.bal_J;
  }
  CUtensorMap tmA, tmB;
  {
    // L per image: {i_h k_w i_c, o_w, i_n} (pitched rows); box = 128 rows or one image slot
    const uint64_t dims[3] = {static_cast<uint64_t>(pl.l_cols), static_cast<uint64_t>(pl.o_w),
                              static_cast<uint64_t>(pl.s.i_n)};
    const uint64_t strides[2] = {static_cast<uint64_t>(pl.pitch) * pl.elt,
                                 static_cast<uint64_t>(pl.pitch) * pl.elt * pl.o_w};
    const uint32_t box[3] = {static_cast<uint32_t>(pl.bk), static_cast<uint32_t>(g.ipt == 1 ? kBM : g.slot),
                             static_cast<uint32_t>(g.ipt)};
    e = encode_tiled(&tmA, tf32, 3, a.L, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(pl.kdim_pad), static_cast<uint64_t>(pl.kc_pad)};
    const uint64_t strides[1] = {static_cast<uint64_t>(pl.kdim_pad) * pl.elt};
    const uint32_t box[2] = {static_cast<uint32_t>(pl.bk), static_cast<uint32_t>(pl.bn / 2)};
    e = encode_tiled(&tmB, tf32, 2, a.Kt, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  CUtensorMap tmB3;
  std::memset(&tmB3, 0, sizeof(tmB3));
  p.b3 = false;
  if (g.b_stream && !(getenv("MEC_PS_B3") && atoi(getenv("MEC_PS_B3")) == 0) && g.aps == 1) {
    // Kt as {kdim_pad, kc_pad, b_open}: the third stride is one window shift
    // (sa atoms); slab z starts z sa atoms further along the same channel row
    // (past a row's end it reads the next row, or the workspace tail reserved
    // for it, Plan::bytes_kt -- never an open row's weights)
    const uint64_t dims[3] = {static_cast<uint64_t>(pl.kdim_pad), static_cast<uint64_t>(pl.kc_pad),
                              static_cast<uint64_t>(g.b_open)};
    const uint64_t strides[2] = {static_cast<uint64_t>(pl.kdim_pad) * pl.elt,
                                 static_cast<uint64_t>(g.sa) * pl.bk * pl.elt};
    const uint32_t box[3] = {static_cast<uint32_t>(pl.bk), static_cast<uint32_t>(pl.bn / 2),
                             static_cast<uint32_t>(g.b_open)};
    if (encode_tiled(&tmB3, tf32, 3, a.Kt, dims, strides, box) == cudaSuccess) p.b3 = true;
    else cudaGetLastError();
  }
  const int64_t pairs = std::min<int64_t>(max_clusters, p.n_items);
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  cfg.numAttrs = getenv("MEC_NO_PDL") ? 1 : 2;
  e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmB3, p);
  if (e != cudaSuccess) return e;
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace mec
