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
//   warp 0     TMA producer: per pipeline stage two K-atoms, each an A window
//              tile (128 rows x 128 B) [+ a B tile (bn rows of Kt x 128 B)
//              when the weights are not resident], 128-byte swizzled,
//              mbarrier complete_tx.
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer: 8 MMAs
//              (M = 128, N = bn, K = 16 bf16 / 8 tf32) per stage wait, with
//              precomputed 32-bit descriptor offsets; fp32 accumulators in
//              TMEM, double-buffered (2 x bn columns) so the epilogue of tile
//              i overlaps the MMAs of tile i+1.
//   warps 2-5  epilogue, one TMEM lane quarter (32 rows) each, in passes of
//              128/64 output bytes per row: tcgen05.ld -> fp32 -> bf16 (RN)
//              or fp32 -> swizzled (conflict-free) shared staging -> one TMA
//              store per image the 32 rows touch.  The box's row coordinate
//              is w = row - n*o_w, so rows outside image n are clipped by the
//              tensor bounds (negative coordinates included): the store
//              writes O[n, h, w, :] directly in n-h-w-c -- for Solution A this
//              applies Alg.2 l.17-19's permutation O[n,h] = O_hnwc[h,n] at
//              store time (MEC_SOLA_FIX_EPILOGUE); with out_hnwc the paper's
//              h-n-w-c intermediate is stored instead.
// Scheduling: the tiles (h, row tile, group, N tile) are split into "combos"
// of one weight variant v = delta(h)/delta_step and one N tile; every CTA
// works on a single combo, so when the combo's weight operand is small
// (bn x kdim_pad, <= 120 KB: C1, C2, C3, ...) it is loaded into shared memory
// ONCE per CTA and stays resident -- only the L windows stream through the
// smem ring.  Within a combo, h is fastest: the CTAs in flight work on
// neighbouring windows of the same L rows (overlapping k_h/s_h-fold), so the
// re-reads hit L2.
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
#include <cstdlib>
#include <cstring>

#include "mec_internal.h"
#include "ptx.cuh"
#include "tma_host.h"

#ifdef MEC_TRACE
// Debug-only stage timestamps (built into a separate libmec_trace.so by
// tools/trace_gemm.py; never in the product library).
__device__ unsigned long long* g_mec_trace = nullptr;
__device__ __forceinline__ unsigned long long mec_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// the buffer pointer is read once per kernel (mec_trace_ptr, a local of the
// kernel): re-reading the __device__ variable per event put a global-load
// latency on every traced step
#define MEC_TRACE_EV(tl, ev)                                                                \
  do {                                                                                      \
    if (mec_trace_ptr != nullptr && (tl) < 64)                                              \
      mec_trace_ptr[(static_cast<size_t>(blockIdx.x) * 64 + (tl)) * 16 + (ev)] = mec_gtime(); \
  } while (0)
// second bank (rows 512 + cta): per-atom builder events
#define MEC_TRACE_EV2(tl, ev)                                                                     \
  do {                                                                                            \
    if (mec_trace_ptr != nullptr && (tl) < 64 && (ev) < 16)                                         \
      mec_trace_ptr[(static_cast<size_t>(blockIdx.x + 512) * 64 + (tl)) * 16 + (ev)] = mec_gtime(); \
  } while (0)
extern "C" int mec_trace_enable(void** dev_buf_out, size_t* bytes_out) {
  const size_t bytes = static_cast<size_t>(1024) * 64 * 16 * 8;
  void* buf = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
  cudaMemset(buf, 0, bytes);
  if (cudaMemcpyToSymbol(g_mec_trace, &buf, sizeof(buf)) != cudaSuccess) return 2;
  *dev_buf_out = buf;
  *bytes_out = bytes;
  return 0;
}
extern "C" int mec_trace_read(void* host, const void* dev, size_t bytes) {
  return cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
}
#else
#define MEC_TRACE_EV(tl, ev) \
  do {                       \
  } while (0)
#define MEC_TRACE_EV2(tl, ev) \
  do {                        \
  } while (0)
#endif

namespace mec {
namespace {

// epilogue warp-groups (alternating tiles): 2 on the TMA paths; 1 on the
// gather path, whose builder warps are the bottleneck (keeps registers unspilled)
template <bool kGather>
constexpr int epi_groups() { return kGather ? 1 : 2; }
constexpr int kBuildGroups = 2;  // gather path: builder warp-groups, atoms dealt round-robin
constexpr int kBuildWarps = 4 * kBuildGroups;  // warps that assemble A atoms in smem
template <bool kGather>
constexpr int kernel_threads() { return 64 + epi_groups<kGather>() * 128 + (kGather ? 32 * kBuildWarps : 0); }
constexpr int kAtomBytes = kBM * kTileKBytes;  // 16 KB: 128 rows x 128 B
constexpr int kMaxAtomsPerStage = 2;
constexpr int kMaxCombos = 32;  // n_var (<= 8) x N tiles (<= 4 for k_c <= 1024)
constexpr int kMaxEpiWarps = 8;

struct GemmParams {
  void* O;
  int64_t o_h, o_w, i_n, k_c;
  // row tiling.  flat: the batch-folded rows n o_w + w in 128-row tiles (one
  // group).  packed: `ipt` images per tile, image j in TMEM lanes
  // [j S, j S + S) (S = o_w rounded up to 32), so no 32-row epilogue block
  // straddles two images; ipt = 1 is one image per tile (Solution B, and
  // Solution A when o_w > 64).
  bool flat;
  bool fused;       // A atoms are TMA boxes of I: atom (a, b, cb) of output row h
  int ncb, k_w, s_h, s_w;
  int pad_h, pad_w;  // fused TMA variant: zero padding through TMA out-of-bounds fill
  // gather path (fused, small i_c): the producer bulk-copies the tile's k_h
  // input rows per image into a 2-slot ring; builder warps assemble each A
  // atom (window elements j = a kwc + r) from them with a per-atom word table
  const unsigned char* gI;   // I base
  const unsigned char* gI_end;
  int k_h;
  int64_t i_h, i_w;
  int row_bytes;    // i_w i_c elt
  int row_pitch;    // staged row pitch (bytes)
  int kwc;          // k_w i_c
  int cpr;          // 16-byte chunks per padded kernel row (kwc_p elt / 16)
  int wstep_b;      // s_w i_c elt
  uint32_t a_col0;  // gather: TMEM column of A stage 0 (after the accumulators)
  uint32_t slot_bytes;
  int n_slots;      // staged-row slots (2..4)
  int ipt, slot;
  int64_t rows, groups, n_mt;
  bool tiles32;     // every tile index fits 32 bits
  int64_t shift;
  int64_t kc_pad;
  int bk;           // K-atom width in elements (64 bf16 / 32 fp32)
  int n_atoms;      // K-atoms per window
  int n_kstages;    // ceil(n_atoms / 2)
  int bn, n_tiles_n;
  int n_var;
  int avec;         // box-start alignment (elements); variant v absorbs delta = h shift mod avec
  int n_combo;      // n_var * n_tiles_n
  int ctas_per_combo;
  int h_first[16];  // smallest h with weight variant v
  // multi-row tiles: a tile computes R consecutive output rows h0 .. h0+R-1;
  // it streams the union of their windows once (columns [h0 shift,
  // (h0+R-1) shift + kdim)) and issues every A atom's MMAs into the R TMEM
  // accumulators it overlaps, B addressed per 32-byte K chunk (needs
  // shift % kchunk == 0, one weight variant, resident weights).  R = 1 is
  // the one-window-per-tile schedule.
  int R;
  int shift_atoms;  // multi-row: shift / bk if a whole number of K-atoms, else 0
  int shift_chunks; // multi-row: shift / kchunk (window start advance per output row, in 32-byte K steps)
  int kchunk;       // elements per 32-byte MMA K step (16 bf16 / 8 tf32)
  int kchunk_log2;
  int n_chunks;     // ceil(kdim / kchunk): B chunks holding weights
  int kdim;
  int stages;
  int aps;          // K-atoms per pipeline stage (2 with resident weights, else 1)
  bool resident;    // weight operand resident in smem
  uint32_t tmem_cols;
  int n_acc;        // TMEM accumulator sets (each R x bn columns)
  uint32_t idesc;
  bool out_hnwc;
  bool tma_store;   // epilogue via TMA stores (k_c elt multiple of 16)
  int pw;           // epilogue pass width (columns); pw * out_elt = 128 / 64 / 32 bytes
  int n_pass;       // bn / pw
  uint32_t stage_out_bytes;  // staging box bytes (32 rows x pw x elt, 1 KB aligned)
  int epi_bufs;              // staging boxes per epilogue warp (1 or 2)
  bool spin;        // gather: builder/MMA handshakes spin on test_wait
  uint32_t backoff_ns;  // gather: nanosleep between probes of the long waits (0 = none)
  int dbg;  // trace builds only: 1 = no epilogue stores, 2 = no MMA, 4 = no A loads,
            // 8 = gather builders skip row loads, 16 = gather builders skip TMEM stores,
            // 64 = epilogue skips TMEM loads
};

struct TileCoord {
  int64_t h, mt, g;  // h = first output row of the tile
  int r_eff;         // output rows in the tile (R, fewer at the end)
  int n_a;           // A atoms streamed for the tile
};

// h-slots of combo v: R == 1: h = h_first[v] + i n_var; R > 1: h0 = i R.
__device__ __forceinline__ int64_t combo_hslots(const GemmParams& p, int v) {
  return p.R == 1 ? (p.o_h - p.h_first[v] + p.n_var - 1) / p.n_var : (p.o_h + p.R - 1) / p.R;
}

// Combo c = v * n_tiles_n + nt.  Tile t of the combo: h-slot fastest, then
// row tile, then group.
__device__ __forceinline__ int64_t combo_tiles(const GemmParams& p, int v) {
  return combo_hslots(p, v) * p.n_mt * p.groups;
}

// nh = combo_hslots(p, v), computed once per CTA
__device__ __forceinline__ TileCoord decode_tile(const GemmParams& p, int v, int64_t nh, int64_t t) {
  TileCoord c;
  int64_t hi;
  if (p.tiles32) {  // 32-bit divisions (tile counts < 2^31): far cheaper than 64-bit ones
    const uint32_t t32 = static_cast<uint32_t>(t), nh32 = static_cast<uint32_t>(nh);
    const uint32_t q = t32 / nh32, nmt = static_cast<uint32_t>(p.n_mt);
    hi = t32 - q * nh32;
    c.mt = q % nmt;
    c.g = q / nmt;
  } else {
    hi = t % nh;
    t /= nh;
    c.mt = t % p.n_mt;
    c.g = t / p.n_mt;
  }
  if (p.R == 1) {
    c.h = p.h_first[v] + hi * p.n_var;
    c.r_eff = 1;
    c.n_a = p.n_atoms;
  } else {
    c.h = hi * p.R;
    c.r_eff = static_cast<int>(min(static_cast<int64_t>(p.R), p.o_h - c.h));
    c.n_a = static_cast<int>(((c.r_eff - 1) * p.shift + p.kdim + p.bk - 1) / p.bk);
  }
  return c;
}

__device__ __noinline__ void p_sink_dummy(uint32_t x) { asm volatile("" ::"r"(x)); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <bool kTF32, bool kGather>
__global__ void __launch_bounds__(kernel_threads<kGather>(), 1)
    window_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmO, const GemmParams p) {
  constexpr int kEpiGroups = epi_groups<kGather>();
  constexpr int kEpiWarps = 4 * kEpiGroups;
  constexpr int kFirstBuildWarp = 2 + kEpiWarps;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
#ifdef MEC_TRACE
  unsigned long long* const mec_trace_ptr = g_mec_trace;
#endif
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + kSmemAlign - 1) & ~uintptr_t(kSmemAlign - 1));
  const int S = p.stages;
  const int kAtomsPerStage = p.aps;
  const int kStageABytes = kAtomsPerStage * kAtomBytes;
  const uint32_t b_tile_bytes = static_cast<uint32_t>(p.bn) * kTileKBytes;
  // smem: [S A-stages][B: n_atoms resident tiles or S x 2 streamed][epi staging][barriers]
  const int nb = p.resident ? p.n_atoms : S * kAtomsPerStage;
  unsigned char* smemA = smem;  // (gather path: A lives in TMEM, no smem ring)
  unsigned char* smemB = smem + (kGather ? 0 : static_cast<size_t>(S) * kStageABytes);
  unsigned char* smemE = smemB + static_cast<size_t>(nb) * b_tile_bytes;
  unsigned char* smemR = smemE + static_cast<size_t>(kEpiWarps) * p.epi_bufs * p.stage_out_bytes;  // gather rows
  uint32_t* ctable = reinterpret_cast<uint32_t*>(smemR + (kGather ? p.n_slots * p.slot_bytes : 0));
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(ctable + (kGather ? p.n_atoms * 8 : 0)) + 15) & ~uintptr_t(15));
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + 4;
  uint64_t* bfull = bars + 2 * S + 8;
  uint64_t* rfull = bars + 2 * S + 9;   // gather row slots (<= 4)
  uint64_t* rempty = bars + 2 * S + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 17);

  // warp index broadcast from lane 0: provably warp-uniform, so role branches
  // are uniform and the MMA issue loop keeps descriptors in uniform registers
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  // this CTA's combo: weight variant v and N tile nt
  const int combo = blockIdx.x % p.n_combo;
  const int v = combo / p.n_tiles_n;
  const int nt = combo % p.n_tiles_n;
  const int64_t t_begin = blockIdx.x / p.n_combo;
  const int64_t t_step = p.ctas_per_combo;
  const int64_t nh_c = combo_hslots(p, v);
  const int64_t n_tiles = nh_c * p.n_mt * p.groups;

  if (warp == 0 && lane == 0) {
    if (!kGather) ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    ptx::tma_prefetch_desc(&tmO);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full[i], kGather ? 4 : 1);  // gather: the 4 warps of one builder group
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&rfull[i], 1);
      ptx::mbar_init(&rempty[i], kBuildWarps);
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 4);  // the 4 warps of one epilogue group
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_dyn(tmem_slot, p.tmem_cols);
  if constexpr (kGather) {
    // staged-row slots start zeroed, so the builders' reads past a staged span
    // (met by zero weight columns) only ever see finite values; chunk table:
    // chunk g of the padded window -> byte offset a row_bytes + 16 (g mod cpr)
    const uint32_t r_s = ptx::smem_u32(smemR);
    for (uint32_t i = threadIdx.x; i < p.n_slots * p.slot_bytes / 16; i += blockDim.x)
      ptx::st_shared_v4(r_s + 16 * i, 0u, 0u, 0u, 0u);
    for (int g = threadIdx.x; g < p.n_atoms * 8; g += blockDim.x) {
      const int a = g / p.cpr, off = g - a * p.cpr;
      ctable[g] = a < p.k_h ? static_cast<uint32_t>(a * p.row_bytes + 16 * off) : 0u;
    }
    ptx::fence_proxy_async_smem();  // zeros before the async-proxy row copies
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) MEC_TRACE_EV(0, 7);
#ifdef MEC_TRACE
  // SM clock check: clock64 and globaltimer at entry and exit (tile slot 62)
  unsigned long long clk0 = 0, gt0 = 0;
  if (threadIdx.x == 0 && mec_trace_ptr != nullptr) {
    clk0 = clock64();
    gt0 = mec_gtime();
  }
#endif
  const int32_t b_row0 = static_cast<int32_t>(v * p.kc_pad + nt * p.bn);

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t hintA = ptx::policy_evict_normal();
      const uint64_t hintB = ptx::policy_evict_last();
      // L and the weight operand come from the preceding kernel (launched as its
      // programmatic dependent): wait for it before the first TMA load.  The
      // gather path's B is loaded by the MMA warp, so its row staging does not wait.
      if (!kGather) ptx::griddep_wait();
      if (!kGather && p.resident && t_begin < n_tiles) {
        ptx::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(p.n_atoms) * b_tile_bytes);
        for (int a = 0; a < p.n_atoms; ++a)
          ptx::tma_load_2d(smemB + static_cast<size_t>(a) * b_tile_bytes, &tmB, bfull, a * p.bk,
                           b_row0, hintB);
      }
      const int64_t kVec = p.avec;  // box-start alignment (elements)
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = t_begin; !kGather && t < n_tiles; t += t_step) {
        const int tl = static_cast<int>((t - t_begin) / t_step);
        MEC_TRACE_EV(tl, 0);
        const TileCoord c = decode_tile(p, v, nh_c, t);
        // window start h*shift rounded down to 16 bytes (TMA rule); variant v absorbs delta
        const int64_t xw = c.h * p.shift;
        const int32_t x0 = static_cast<int32_t>(xw - xw % kVec);
        const int32_t y0 = static_cast<int32_t>(c.mt * kBM);
        const int32_t z0 = static_cast<int32_t>(c.g);
        const int n_ks = (c.n_a + kAtomsPerStage - 1) / kAtomsPerStage;
        for (int ks = 0; ks < n_ks; ++ks) {
          const int na = min(kAtomsPerStage, c.n_a - ks * kAtomsPerStage);
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (p.dbg & 4) {
            ptx::mbar_arrive(&full[stage]);
          } else {
            ptx::mbar_arrive_expect_tx(
                &full[stage], static_cast<uint32_t>(na) * (kAtomBytes + (p.resident ? 0u : b_tile_bytes)));
            for (int a = 0; a < na; ++a) {
              const int atom = ks * kAtomsPerStage + a;
              unsigned char* dstA = smemA + static_cast<size_t>(stage) * kStageABytes + a * kAtomBytes;
              if (p.fused) {
                // K atom -> (kernel row a, kernel column b, channel block cb); rows = pixels
                // s_w w + b of input row s_h h + a (pixel traversal stride s_w in the map)
                const int ab = atom / p.ncb, cb = atom - ab * p.ncb;
                const int fa = ab / p.k_w, fb = ab - fa * p.k_w;
                // zero padding (NEXT-4): coordinates of the unpadded I, shifted by the
                // pads; TMA zero-fills the out-of-bounds pixels and rows of a box
                const int32_t zy = static_cast<int32_t>(c.h * p.s_h + fa - p.pad_h);
                if (p.ipt <= 1) {
                  ptx::tma_load_4d(dstA, &tmA, &full[stage], cb * p.bk,
                                   static_cast<int32_t>(c.mt * kBM * p.s_w + fb - p.pad_w), zy, z0, hintA);
                } else {
                  for (int j = 0; j < p.ipt; ++j)
                    ptx::tma_load_4d(dstA + j * p.slot * kTileKBytes, &tmA, &full[stage], cb * p.bk,
                                     fb - p.pad_w, zy, z0 * p.ipt + j, hintA);
                }
              } else if (p.ipt <= 1) {
                ptx::tma_load_3d(dstA, &tmA, &full[stage], x0 + atom * p.bk, y0, z0, hintA);
              } else {  // one box of `slot` rows per image of the tile (images >= i_n: zero fill)
                for (int j = 0; j < p.ipt; ++j)
                  ptx::tma_load_3d(dstA + j * p.slot * kTileKBytes, &tmA, &full[stage],
                                   x0 + atom * p.bk, 0, z0 * p.ipt + j, hintA);
              }
              if (!p.resident)
                ptx::tma_load_2d(smemB + static_cast<size_t>(stage * kAtomsPerStage + a) * b_tile_bytes,
                                 &tmB, &full[stage], atom * p.bk, b_row0, hintB);
            }
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        MEC_TRACE_EV(tl, 1);
      }
    }
    if constexpr (kGather) {
      // Stage the k_h input rows s_h h + a of each image of the tile.  They are
      // contiguous in I: one bulk copy per image (lane j copies image j) of the
      // span's 16-byte-aligned superset; the builders recompute its offset.  A
      // tile's coordinates and copy sizes are computed before waiting for its
      // slot, so that arithmetic overlaps the wait.
      const uintptr_t iend = reinterpret_cast<uintptr_t>(p.gI_end);
      const uint32_t span = static_cast<uint32_t>(p.k_h * p.row_bytes);
      for (int64_t t = t_begin; t < n_tiles; t += t_step) {
        const int tl = static_cast<int>((t - t_begin) / t_step);
        const int slotid = tl % p.n_slots;
        const TileCoord c = decode_tile(p, v, nh_c, t);
        const int64_t n = c.g * p.ipt + lane;
        const bool mine = lane < p.ipt && n < p.i_n;
        uintptr_t s0 = 0, s1 = 0, tail0 = 0;
        if (mine) {
          const uintptr_t src = reinterpret_cast<uintptr_t>(p.gI) +
                                static_cast<uintptr_t>((n * p.i_h + c.h * p.s_h) * p.row_bytes);
          s0 = src & ~uintptr_t(15);
          s1 = (src + span + 15) & ~uintptr_t(15);
          // the very end of I may fall inside a 16-byte granule: bulk-copy up to the
          // last full granule, the final bytes with plain loads
          tail0 = s1 > iend ? (iend & ~uintptr_t(15)) : s1;
        }
        const uint32_t bytes = __reduce_add_sync(0xffffffffu, static_cast<uint32_t>(tail0 - s0));
        unsigned char* dimg = smemR + static_cast<size_t>(slotid) * p.slot_bytes +
                              static_cast<size_t>(lane) * p.k_h * p.row_pitch;
        if (p.backoff_ns > 0) ptx::mbar_wait_backoff(&rempty[slotid], ((tl / p.n_slots) & 1) ^ 1, p.backoff_ns);
        else ptx::mbar_wait(&rempty[slotid], ((tl / p.n_slots) & 1) ^ 1);
        if (lane == 0) MEC_TRACE_EV(tl, 7);
        if (mine && tail0 < s1) {
          for (uintptr_t b = tail0; b < iend && b < s1; ++b)
            dimg[b - s0] = *reinterpret_cast<const unsigned char*>(b);
          __threadfence_block();
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_expect_tx(&rfull[slotid], bytes);  // release: tails above
        __syncwarp();
        if (mine && tail0 > s0)
          ptx::bulk_load(dimg, reinterpret_cast<const void*>(s0), static_cast<uint32_t>(tail0 - s0),
                         &rfull[slotid]);
        if (lane == 0) MEC_TRACE_EV(tl, 15);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    int stage = 0;
    uint32_t phase = 0;
    const uint64_t a_desc0 = ptx::smem_desc_sw128(ptx::smem_u32(smemA));
    const uint64_t b_desc0 = ptx::smem_desc_sw128(ptx::smem_u32(smemB));
    const uint32_t b_tile16 = b_tile_bytes >> 4;
    if (kGather && p.resident && t_begin < n_tiles && lane == 0) {
      // gather path: the resident weights (prepared by the preceding kernel) are
      // loaded here, after the grid dependency, while the producer stages rows
      ptx::griddep_wait();
      ptx::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(p.n_atoms) * b_tile_bytes);
      for (int a = 0; a < p.n_atoms; ++a)
        ptx::tma_load_2d(smemB + static_cast<size_t>(a) * b_tile_bytes, &tmB, bfull, a * p.bk, b_row0,
                         ptx::policy_evict_last());
    }
    if (p.resident && t_begin < n_tiles) ptx::mbar_wait(bfull, 0);
    for (int64_t t = t_begin; t < n_tiles; t += t_step) {
      const int tl = static_cast<int>((t - t_begin) / t_step);
      const TileCoord c = decode_tile(p, v, nh_c, t);
      const int acc = tl % p.n_acc;
      const uint32_t acc_phase = static_cast<uint32_t>(tl / p.n_acc) & 1u;
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      if (lane == 0) MEC_TRACE_EV(tl, 2);
      const uint32_t d_set = tmem_base + static_cast<uint32_t>(acc * p.R * p.bn);
      const int n_ks = (c.n_a + kAtomsPerStage - 1) / kAtomsPerStage;
      for (int ks = 0; ks < n_ks; ++ks) {
        const int na = min(kAtomsPerStage, c.n_a - ks * kAtomsPerStage);
        if (kGather && p.spin) ptx::mbar_spin(&full[stage], phase);
        else if (!(p.dbg & 128)) ptx::mbar_wait(&full[stage], phase);  // (trace builds: 128 = no full waits)
        ptx::tc_fence_after();
        if (ks == 0 && lane == 0) MEC_TRACE_EV(tl, 3);
        if (kGather && ks < 7 && lane == 0) MEC_TRACE_EV(tl, 8 + ks);
        {
          // the whole warp runs the (warp-uniform) descriptor arithmetic; one
          // elected lane issues each MMA / commit
          const uint32_t a_off = static_cast<uint32_t>(stage * kStageABytes) >> 4;
          if constexpr (kGather) {
            // A atom in TMEM columns a_col0 + 32 stage .. + 31: 4 MMAs of K = 32 bytes
            const uint32_t a_tm = tmem_base + p.a_col0 + static_cast<uint32_t>(stage * 32);
            const uint64_t bd = b_desc0 + static_cast<uint32_t>(ks) * b_tile16;
            if (!(p.dbg & 2)) ptx::mma_ts_atom_elect<kTF32>(d_set, a_tm, bd, p.idesc, ks != 0 ? 1u : 0u);
          }
          for (int a = 0; !kGather && a < na; ++a) {
            const uint64_t ad = a_desc0 + a_off + static_cast<uint32_t>(a * (kAtomBytes >> 4));
            if (p.R == 1) {
              const uint32_t b_atom = p.resident ? static_cast<uint32_t>(ks * kAtomsPerStage + a)
                                                 : static_cast<uint32_t>(stage * kAtomsPerStage + a);
              const uint64_t bd = b_desc0 + b_atom * b_tile16;
#pragma unroll
              for (int k = 0; k < 4; ++k) {  // 4 x 32 B = one 128-byte atom row
                if (p.dbg & 2) break;
                ptx::mma_ss_elect<kTF32>(d_set, ad + 2 * k, bd + 2 * k, p.idesc,
                                         (ks | a | k) != 0 ? 1u : 0u);
              }
            } else {
              // multi-row tile (shift a multiple of the K-atom): stream atom
              // (ks aps + a) is atom  b = stream atom - r shift_atoms  of output
              // row h0 + r's window -- the same 4 MMAs as R = 1, into
              // accumulator r against resident weight tile b
              const int sa = ks * kAtomsPerStage + a;
              if (p.shift_atoms > 0) {
                for (int r = 0; r < c.r_eff; ++r) {
                  const int b = sa - r * p.shift_atoms;
                  if (b < 0 || b >= p.n_atoms || (p.dbg & 2)) continue;
                  ptx::mma_ss_atom_elect<kTF32>(d_set + static_cast<uint32_t>(r * p.bn), ad,
                                                b_desc0 + static_cast<uint32_t>(b) * b_tile16, p.idesc,
                                                b != 0 ? 1u : 0u);
                }
              } else {
                // shift a whole 32-byte K step only: the atom's K step k meets
                // B chunk c0 + k of row r (chunk = 32 bytes of a B tile row)
                const int nbc = 4 * p.n_atoms;
                for (int r = 0; r < c.r_eff; ++r) {
                  const int c0 = 4 * sa - r * p.shift_chunks;
                  if (c0 + 3 < 0 || c0 >= nbc || (p.dbg & 2)) continue;
                  const uint32_t d = d_set + static_cast<uint32_t>(r * p.bn);
                  auto bdesc = [&](int ch) -> uint64_t {
                    return b_desc0 + static_cast<uint32_t>((ch >> 2) * static_cast<int>(b_tile16) + (ch & 3) * 2);
                  };
                  if (c0 >= 0 && c0 + 3 < nbc) {
                    ptx::mma_ss_atom4b_elect<kTF32>(d, ad, bdesc(c0), bdesc(c0 + 1), bdesc(c0 + 2), bdesc(c0 + 3),
                                                    p.idesc, c0 != 0 ? 1u : 0u);
                  } else {
                    for (int k = 0; k < 4; ++k) {
                      const int ch = c0 + k;
                      if (ch < 0 || ch >= nbc) continue;
                      ptx::mma_ss_elect<kTF32>(d, ad + 2 * k, bdesc(ch), p.idesc, ch != 0 ? 1u : 0u);
                    }
                  }
                }
              }
            }
          }
          ptx::mma_commit_elect(&empty[stage]);
          if (ks == n_ks - 1) {
            ptx::mma_commit_elect(&tfull[acc]);
            if (lane == 0) MEC_TRACE_EV(tl, 4);
          }
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (kGather && warp >= kFirstBuildWarp) {
    // ===================== A-atom builders (gather path) =====================
    // Thread (quarter q = warp % 4, lane) owns tile row m = 32 q + lane: output
    // pixel w of image slot j.  An A atom is 128 bytes of that row's padded
    // window = 8 chunks of 16 bytes; chunk g is the contiguous run of I at
    // staged byte  base(j) + w wstep_b + ctable[g]  (ctable: a row_bytes +
    // 16 (g mod cpr)).  The atom goes to TMEM (tcgen05.st, row m -> lane m),
    // where the MMA reads it as its A operand.  Builder group bgroup builds
    // atoms bgroup, bgroup + kBuildGroups, ... of every tile.
    const int wbg = warp - kFirstBuildWarp;
    const int quarter = warp & 3;             // TMEM lanes [32 quarter, 32 quarter + 32)
    const int bgroup = wbg >> 2;
    const uint32_t table_s = ptx::smem_u32(ctable);
    const uint32_t r_smem = ptx::smem_u32(smemR);
    const uint32_t t_row = tmem_base + (static_cast<uint32_t>(32 * quarter) << 16) + p.a_col0;
    const int m = 32 * quarter + lane;
    // image slot of this row (rows past ipt slots -- fewer images than the tile
    // holds -- read slot 0's data and are never stored)
    const int j = m / p.slot < p.ipt ? m / p.slot : 0;
    const int w_last = static_cast<int>(p.o_w) - 1;
    // global atom sequence number: stage = seq mod S (S a power of two on this
    // path); group g builds the atoms with seq = g mod kBuildGroups (balanced
    // even when n_atoms is odd)
    uint32_t seq = 0, seq_mod = 0;  // seq_mod = seq mod kBuildGroups
    const uint32_t s_mask = static_cast<uint32_t>(S - 1);
    const int s_log2 = __ffs(S) - 1;
    for (int64_t t = t_begin; t < n_tiles; t += t_step) {
      const int tl = static_cast<int>((t - t_begin) / t_step);
      const int slotid = tl % p.n_slots;
      const TileCoord c = decode_tile(p, v, nh_c, t);
      const int w = min(static_cast<int>(c.mt * kBM) + m - j * p.slot, w_last);
      const int64_t n = c.g * p.ipt + j;
      // offset of the image's span inside its 16-byte-aligned bulk copy
      const uint32_t sh = n < p.i_n ? static_cast<uint32_t>((reinterpret_cast<uintptr_t>(p.gI) +
                                                              static_cast<uintptr_t>((n * p.i_h + c.h * p.s_h) * p.row_bytes)) & 15)
                                    : 0u;
      const uint32_t base = r_smem + static_cast<uint32_t>(slotid) * p.slot_bytes +
                            static_cast<uint32_t>(j * p.k_h * p.row_pitch) + sh +
                            static_cast<uint32_t>(w * p.wstep_b);
      ptx::mbar_wait(&rfull[slotid], (tl / p.n_slots) & 1);
      if (wbg == 0 && lane == 0) MEC_TRACE_EV(tl, 0);
      const int atom0 = static_cast<int>((static_cast<uint32_t>(bgroup) + kBuildGroups - seq_mod) % kBuildGroups);
      for (int atom = atom0; atom < p.n_atoms; atom += kBuildGroups) {
        const uint32_t aseq = seq + static_cast<uint32_t>(atom);
        const int stage = static_cast<int>(aseq & s_mask);
        const uint32_t phase = (aseq >> s_log2) & 1u;
        // two halves of 4 chunks (64 bytes of the row): all of a half's loads
        // first (the asm loads keep program order, so interleaving them with the
        // shifts would serialise their latencies), then its shifts and a
        // 16-column TMEM store
        const uint32_t t_atom = t_row + static_cast<uint32_t>(stage * 32);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint4 tt = ptx::ld_shared_v4(table_s + static_cast<uint32_t>(atom * 32 + half * 16));
          const uint32_t addr[4] = {base + tt.x, base + tt.y, base + tt.z, base + tt.w};
          uint2 xs[4][3];
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            const uint32_t al = addr[ch] & ~7u;
#ifdef MEC_TRACE
            if (p.dbg & 8) {  // trace builds: no row loads
              xs[ch][0] = xs[ch][1] = xs[ch][2] = make_uint2(al, al);
              continue;
            }
#endif
            xs[ch][0] = ptx::ld_shared_v2(al);
            xs[ch][1] = ptx::ld_shared_v2(al + 8);
            xs[ch][2] = ptx::ld_shared_v2(al + 16);
          }
          uint32_t val[16];
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            const uint32_t A = addr[ch];
            const uint2 x0 = xs[ch][0], x1 = xs[ch][1], x2 = xs[ch][2];
            const bool hi = (A & 4u) != 0;
            const uint32_t w0 = hi ? x0.y : x0.x, w1 = hi ? x1.x : x0.y, w2 = hi ? x1.y : x1.x;
            const uint32_t w3 = hi ? x2.x : x1.y, w4 = hi ? x2.y : x2.x;
            const uint32_t bs = A << 3;  // shf.r uses the low 5 bits: (A mod 4) bytes
            val[4 * ch + 0] = __funnelshift_r(w0, w1, bs);
            val[4 * ch + 1] = __funnelshift_r(w1, w2, bs);
            val[4 * ch + 2] = __funnelshift_r(w2, w3, bs);
            val[4 * ch + 3] = __funnelshift_r(w3, w4, bs);
          }
          if (half == 0) {
            if (p.spin) ptx::mbar_spin(&empty[stage], phase ^ 1);  // the MMAs that read this stage are done
            else ptx::mbar_wait(&empty[stage], phase ^ 1);
            ptx::tc_fence_after();
          }
#ifdef MEC_TRACE
          if (p.dbg & 16) {  // trace builds: 16 = no TMEM stores
            uint32_t acc = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) acc ^= val[i];
            if (acc == 0x12345678u) p_sink_dummy(acc);
            continue;
          }
#endif
          ptx::tmem_st_32x32b_x16(t_atom + static_cast<uint32_t>(16 * half), val);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&full[stage]);
        if (lane == 0 && atom < 4) MEC_TRACE_EV2(tl, quarter * 4 + atom);
      }
      seq += static_cast<uint32_t>(p.n_atoms);
      seq_mod = (seq_mod + static_cast<uint32_t>(p.n_atoms)) % kBuildGroups;
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&rempty[slotid]);
      if (wbg == 0 && lane == 0) MEC_TRACE_EV(tl, 1);
    }
  } else {
    // ===================== epilogue (warps 2..9: two groups) =====================
    const int quarter = warp & 3;  // TMEM lanes [32 quarter, 32 quarter + 32)
    const int group = (warp - 2) >> 2;  // group g takes tiles tl = g, g + 2, ...
    constexpr int kOutElt = kTF32 ? 4 : 2;
    // per-warp staging: epi_bufs boxes used in turn, so a pass does not wait for
    // the previous pass's TMA store to finish reading its box
    unsigned char* const stg_gen0 = smemE + static_cast<size_t>(warp - 2) * p.epi_bufs * p.stage_out_bytes;
    const uint32_t stg0 = ptx::smem_u32(stg_gen0);
    int ebuf = 0;
    const int row_bytes = p.pw * kOutElt;  // 128, 64 or 32
    // swizzle of the staging box (matches the O tensor map): chunk c of row r
    // lives at chunk c ^ f(r) -- conflict-free 16-byte stores
    const int swz_shift = row_bytes == 128 ? 0 : (row_bytes == 64 ? 1 : 2);
    const int swz_mask = row_bytes == 128 ? 7 : (row_bytes == 64 ? 3 : 1);
    const uint32_t my_x = static_cast<uint32_t>((lane >> swz_shift) & swz_mask);
    const int64_t cols_left = p.k_c - static_cast<int64_t>(nt) * p.bn;
    for (int64_t t = t_begin + group * t_step; t < n_tiles; t += kEpiGroups * t_step) {
      const int tl = static_cast<int>((t - t_begin) / t_step);
      const int acc = tl % p.n_acc;
      const uint32_t acc_phase = static_cast<uint32_t>(tl / p.n_acc) & 1u;
      TileCoord c = decode_tile(p, v, nh_c, t);
      // this warp's 32 rows: image n, columns w0 .. w0 + nvalid - 1 (packed), or
      // flattened rows gr0 .. gr0 + nvalid - 1 (flat)
      int64_t gr0, nvalid, n_img = 0, w0 = 0;
      if (p.flat) {
        const int64_t r0 = c.mt * kBM + quarter * 32;
        nvalid = min(static_cast<int64_t>(32), p.rows - r0);
        gr0 = r0;
      } else {
        const int j = (quarter * 32) / p.slot;
        n_img = c.g * p.ipt + j;
        w0 = c.mt * kBM + quarter * 32 - j * p.slot;
        nvalid = (j < p.ipt && n_img < p.i_n) ? min(static_cast<int64_t>(32), p.o_w - w0) : 0;
        gr0 = n_img * p.o_w + w0;
      }
      // this lane's output row: O[n, h, w] (or O_hnwc[h, n o_w + w]) at column nt*bn
      unsigned char* orow_own;
      {
        const int64_t gr = gr0 + lane;
        int64_t out_row;
        if (p.out_hnwc) {
          out_row = c.h * (p.i_n * p.o_w) + gr;
        } else if (p.tiles32) {  // (i_n o_w < 2^31 too: a 32-bit division)
          const int64_t n = static_cast<uint32_t>(gr) / static_cast<uint32_t>(p.o_w), w = gr - n * p.o_w;
          out_row = (n * p.o_h + c.h) * p.o_w + w;
        } else {
          const int64_t n = gr / p.o_w, w = gr - n * p.o_w;
          out_row = (n * p.o_h + c.h) * p.o_w + w;
        }
        orow_own = static_cast<unsigned char*>(p.O) +
                   (out_row * p.k_c + static_cast<int64_t>(nt) * p.bn) * kOutElt;
      }
      if (p.backoff_ns > 0) ptx::mbar_wait_backoff(&tfull[acc], acc_phase, p.backoff_ns);
      else ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      if ((warp & 3) == 2 && lane == 0) MEC_TRACE_EV(tl, 5);
      const int64_t h_tile = c.h;
      for (int rr = 0; rr < c.r_eff; ++rr) {
      c.h = h_tile + rr;  // output row stored by this sub-pass
      if (rr > 0) orow_own += (p.out_hnwc ? p.i_n * p.o_w : p.o_w) * p.k_c * kOutElt;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                             static_cast<uint32_t>((acc * p.R + rr) * p.bn);
      for (int pass = 0; pass < p.n_pass; ++pass) {
        const int c0 = pass * p.pw;
        uint32_t v16[4][16];
#pragma unroll
        if (p.dbg & 64) {  // trace builds: no TMEM loads in the epilogue
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 16; ++e) v16[j][e] = static_cast<uint32_t>(c0 + e);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j * 16 < p.pw) ptx::tmem_ld_32x32b_x16(taddr + c0 + 16 * j, v16[j]);
          ptx::tmem_ld_wait();
        }
        if (!kGather && (warp & 3) == 2 && lane == 0 && pass < 2) MEC_TRACE_EV(tl, 8 + 4 * pass);
        if (nvalid <= 0 || c0 >= cols_left) continue;  // warp-uniform
        if (p.tma_store) {
          // the TMA store that last used this staging box must have finished reading it
          const uint32_t stg = stg0 + static_cast<uint32_t>(ebuf) * p.stage_out_bytes;
          unsigned char* const stg_gen = stg_gen0 + static_cast<size_t>(ebuf) * p.stage_out_bytes;
          const uint32_t my_row = stg + static_cast<uint32_t>(lane * row_bytes);
          if (++ebuf == p.epi_bufs) ebuf = 0;
          if (lane == 0) {
            if (p.epi_bufs > 1)
              ptx::bulk_wait_group_read<1>();
            else
              ptx::bulk_wait_group_read<0>();
          }
          __syncwarp();
          if (!kGather && (warp & 3) == 2 && lane == 0 && pass < 2) MEC_TRACE_EV(tl, 10 + 4 * pass);
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
              q0 = pack_bf16x2(__uint_as_float(v16[j][e]), __uint_as_float(v16[j][e + 1]));
              q1 = pack_bf16x2(__uint_as_float(v16[j][e + 2]), __uint_as_float(v16[j][e + 3]));
              q2 = pack_bf16x2(__uint_as_float(v16[j][e + 4]), __uint_as_float(v16[j][e + 5]));
              q3 = pack_bf16x2(__uint_as_float(v16[j][e + 6]), __uint_as_float(v16[j][e + 7]));
            }
            ptx::st_shared_v4(my_row + ((static_cast<uint32_t>(ch) ^ my_x) << 4), q0, q1, q2, q3);
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (!kGather && (warp & 3) == 2 && lane == 0 && pass < 2) MEC_TRACE_EV(tl, 9 + 4 * pass);
          const int32_t col = static_cast<int32_t>(nt * p.bn + c0);
          if (!p.flat) {
            // packed: the 32 rows lie in image n_img (rows past o_w are clipped)
            if (lane == 0 && !(p.dbg & 1)) {
              if (p.out_hnwc)  // O_hnwc as {k_c, o_w, i_n, o_h}
                ptx::tma_store_4d(&tmO, stg_gen, col,
                                  static_cast<int32_t>(w0), static_cast<int32_t>(n_img),
                                  static_cast<int32_t>(c.h));
              else  // O as {k_c, o_w, o_h, i_n}
                ptx::tma_store_4d(&tmO, stg_gen, col,
                                  static_cast<int32_t>(w0), static_cast<int32_t>(c.h),
                                  static_cast<int32_t>(n_img));
              ptx::bulk_commit_group();
            }
          } else if (p.out_hnwc) {
            if (lane == 0 && !(p.dbg & 1)) {
              ptx::tma_store_3d(&tmO, stg_gen, col,
                                static_cast<int32_t>(gr0), static_cast<int32_t>(c.h));
              ptx::bulk_commit_group();
            }
          } else {
            // rows of the first image: one TMA store (rows past o_w are clipped);
            // TMA stores reject negative coordinates, so the rows of any later
            // image in this 32-row block are stored from the staging box by the
            // warp (16 B per lane, coalesced)
            const int64_t n_first = gr0 / p.o_w;
            const int k_first = static_cast<int>(min(nvalid, (n_first + 1) * p.o_w - gr0));
            if (lane == 0 && !(p.dbg & 1)) {
              ptx::tma_store_4d(&tmO, stg_gen, col,
                                static_cast<int32_t>(gr0 - n_first * p.o_w), static_cast<int32_t>(c.h),
                                static_cast<int32_t>(n_first));
              ptx::bulk_commit_group();
            }
            if (k_first < nvalid && !(p.dbg & 1)) {
              const int lg = nchunk == 8 ? 3 : (nchunk == 4 ? 2 : 1);
              const int nrest = static_cast<int>(nvalid) - k_first;
              const int total = nrest * nchunk;
              for (int ci0 = 0; ci0 < total; ci0 += 32) {  // warp-uniform trip count
                const int ci = min(ci0 + lane, total - 1);
                const int row = k_first + (ci >> lg), ch = ci & (nchunk - 1);
                const unsigned long long base =
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(orow_own), row);
                const uint32_t x = static_cast<uint32_t>((row >> swz_shift) & swz_mask);
                const uint4 val = ptx::ld_shared_v4(stg + static_cast<uint32_t>(row * row_bytes) +
                                                    ((static_cast<uint32_t>(ch) ^ x) << 4));
                if (ci0 + lane < total)
                  *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(base) + c0 * kOutElt + ch * 16) =
                      val;
              }
            }
          }
        } else if (lane < nvalid) {
          // k_c * elt not a multiple of 16 (or k_c not a multiple of the pass
          // width): element stores from registers
          unsigned char* orow = orow_own;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int col = c0 + j * 16 + e;
              if (j * 16 + e < p.pw && col < cols_left) {
                if constexpr (kTF32) {
                  reinterpret_cast<uint32_t*>(orow)[col] = v16[j][e];
                } else {
                  const uint32_t pkd = pack_bf16x2(__uint_as_float(v16[j][e]), 0.0f);
                  reinterpret_cast<uint16_t*>(orow)[col] = static_cast<uint16_t>(pkd & 0xFFFFu);
                }
              }
            }
          }
        }
      }
      }  // rows rr of the tile
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      if ((warp & 3) == 2 && lane == 0) MEC_TRACE_EV(tl, 6);
    }
    if (lane == 0) ptx::bulk_wait_group<0>();
  }

  ptx::tc_fence_before();
  __syncthreads();
#ifdef MEC_TRACE
  if (threadIdx.x == 0 && mec_trace_ptr != nullptr) {
    unsigned long long* c = mec_trace_ptr + (static_cast<size_t>(blockIdx.x) * 64 + 62) * 16;
    c[0] = clk0;
    c[1] = clock64();
    c[2] = gt0;
    c[3] = mec_gtime();
  }
#endif
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

}  // namespace

bool fused_eligible(const Plan& pl) {
  return (pl.s.i_c * pl.elt) % kTileKBytes == 0 && pl.s_w <= 2;
}

namespace {
// staged row pitch: row bytes + slack for the 16-byte alignment shift of a
// span and the builders' 24-byte chunk reads past its end
int gather_row_pitch(const Plan& pl) {
  return static_cast<int>((pl.s.i_w * pl.s.i_c * pl.elt + 48 + 15) / 16 * 16);
}
int tile_ipt(const Plan& pl) {
  if (pl.o_w > 128) return 1;
  const int slot = static_cast<int>((pl.o_w + 31) / 32 * 32);
  return std::max(1, 128 / slot);
}
int64_t gather_slot_bytes(const Plan& pl, int ipt) {
  return (static_cast<int64_t>(ipt) * pl.s.k_h * gather_row_pitch(pl) + 127) / 128 * 128;
}
constexpr size_t kSmemBudget = 222 * 1024;  // usable dynamic smem after the 1 KB alignment slack
// epilogue staging boxes (32 rows x 128/64/32 bytes) per epilogue warp: 2 on
// the gather path (4 epilogue warps), 1 on the TMA paths (8 warps; their smem
// goes to A stages)
int epi_bufs(bool gather) { return gather ? 2 : 1; }
size_t epi_bytes(const Plan& pl, bool gather) {
  int row_bytes = 128;
  while (row_bytes > 32 && (pl.bn * pl.elt) % row_bytes != 0) row_bytes /= 2;
  return static_cast<size_t>(4 * (gather ? 1 : 2)) * epi_bufs(gather) * 32 * row_bytes;
}
// gather path: images per tile -- as many as the 128 rows hold, fewer when two
// staged-row slots would not fit next to the resident weights (large strides:
// many images of few output pixels, each needing k_h input rows); 0 = none fits
int gather_ipt(const Plan& pl) {
  const int64_t n_atoms = pl.kdim_g / pl.bk;
  const int64_t fixed = static_cast<int64_t>(pl.bn) * kTileKBytes * n_atoms + n_atoms * 32 + 64 +
                        static_cast<int64_t>(epi_bytes(pl, true));
  for (int ipt = tile_ipt(pl); ipt >= 1; --ipt)
    if (fixed + 2 * gather_slot_bytes(pl, ipt) <= static_cast<int64_t>(kSmemBudget)) return ipt;
  return 0;
}
}  // namespace

bool gather_eligible(const Plan& pl) {
  if (fused_eligible(pl)) return false;
  // one N tile (k_c <= 256); weights resident next to two staged-row slots; A in TMEM;
  // unpadded input (the staged rows are copied verbatim)
  return pl.n_tiles_n == 1 && gather_ipt(pl) > 0 && pl.pad_h == 0 && pl.pad_w == 0 && pl.s.i_w * pl.s.i_c * pl.elt < (1LL << 24) &&
         pl.s.k_h < 256;
}

cudaError_t launch_window_gemm(const Plan& pl, const GemmArgs& a, cudaStream_t st,
                               int* launches) {
  const bool tf32 = pl.dt == MEC_DTYPE_TF32;
  const int out_elt = pl.elt;
  CUtensorMap tmA, tmB, tmO;
  // Row tiling (see GemmParams): Solution A with o_w < 32 folds flat (a
  // 32-row epilogue block then spans several images); otherwise image slots.
  // (as the h-sweep: flat rows also for o_w <= 64 with a 16-byte aligned
  // window shift; MEC_SWEEP_FLAT64=0: image slots)
  const bool flat64 = pl.o_w <= 64 && pl.shift % (16 / pl.elt) == 0 &&
                      !(getenv("MEC_SWEEP_FLAT64") && atoi(getenv("MEC_SWEEP_FLAT64")) == 0);
  const bool flat = !a.fused && a.batch_folded && (pl.o_w < 32 || flat64);
  int slot = 128, ipt = 1;
  const bool gather = a.fused && !fused_eligible(pl);
  if (!flat && pl.o_w <= 128) {
    slot = static_cast<int>((pl.o_w + 31) / 32 * 32);
    if (a.batch_folded) ipt = std::max(1, 128 / slot);
    if (gather) ipt = gather_ipt(pl);  // fewer when the staged rows would not fit
    if (ipt < 1) return cudaErrorInvalidConfiguration;
    if (ipt == 1) slot = 128;
  }
  const int64_t rows = flat ? pl.s.i_n * pl.o_w : pl.o_w;
  const int64_t groups = flat ? 1 : (pl.s.i_n + ipt - 1) / ipt;
  const int64_t n_mt = flat ? (rows + kBM - 1) / kBM : (ipt > 1 ? 1 : (pl.o_w + kBM - 1) / kBM);
  if (gather) {
    std::memset(&tmA, 0, sizeof(tmA));  // A atoms are assembled in smem by builder warps
  } else if (a.fused) {
    // A: the NHWC input as {i_c, i_w, i_h, i_n}; a box is bk channels x `rows`
    // pixels taken every s_w pixels (elementStrides) -- one K-atom of `rows`
    // windows, read in place: L is never materialised.
    // (the caller's unpadded I: src_w x src_h pixels)
    const uint64_t dims[4] = {static_cast<uint64_t>(pl.s.i_c), static_cast<uint64_t>(pl.src_w),
                              static_cast<uint64_t>(pl.src_h), static_cast<uint64_t>(pl.s.i_n)};
    const uint64_t strides[3] = {static_cast<uint64_t>(pl.s.i_c) * pl.elt,
                                 static_cast<uint64_t>(pl.src_w * pl.s.i_c) * pl.elt,
                                 static_cast<uint64_t>(pl.src_h * pl.src_w * pl.s.i_c) * pl.elt};
    const uint32_t rows_box = static_cast<uint32_t>(ipt > 1 ? slot : kBM);
    const uint32_t box[4] = {static_cast<uint32_t>(pl.bk), rows_box * static_cast<uint32_t>(pl.s_w), 1, 1};
    const uint32_t es[4] = {1, static_cast<uint32_t>(pl.s_w), 1, 1};
    cudaError_t e = encode_tiled_strided(&tmA, tf32, 4, a.L, dims, strides, box, es);
    if (e != cudaSuccess) return e;
  } else
  // A: the lowered tensor L (Alg.2 l.9 / l.21) as {columns, rows, groups}:
  // flat {i_h k_w i_c, i_n o_w, 1}, else per image {i_h k_w i_c, o_w, i_n}.
  {
    const uint64_t dims[3] = {static_cast<uint64_t>(pl.l_cols), static_cast<uint64_t>(rows),
                              static_cast<uint64_t>(flat ? 1 : pl.s.i_n)};
    const uint64_t strides[2] = {static_cast<uint64_t>(pl.pitch) * pl.elt,
                                 static_cast<uint64_t>(pl.pitch) * pl.elt * rows};
    const uint32_t box[3] = {static_cast<uint32_t>(pl.bk), static_cast<uint32_t>(ipt > 1 ? slot : kBM), 1};
    cudaError_t e = encode_tiled(&tmA, tf32, 3, a.L, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  // B: the prepared weight operand Kt, n_var x kc_pad rows of kdim_pad, K-major.
  {
    const int64_t kcols = gather ? pl.kdim_g : pl.kdim_pad;
    const uint64_t dims[2] = {static_cast<uint64_t>(kcols),
                              static_cast<uint64_t>((gather ? 1 : pl.n_var) * pl.kc_pad)};
    const uint64_t strides[1] = {static_cast<uint64_t>(kcols) * pl.elt};
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
  p.flat = flat;
  p.ipt = ipt;
  p.slot = slot;
  p.rows = rows;
  p.groups = groups;
  p.n_mt = n_mt;
  p.shift = pl.shift;
  p.kc_pad = pl.kc_pad;
  p.bk = pl.bk;
  p.n_atoms = static_cast<int>(gather ? pl.kdim_g / pl.bk
                                      : (a.fused ? (pl.kdim + pl.bk - 1) / pl.bk : pl.kdim_pad / pl.bk));
  p.cpr = static_cast<int>(pl.kwc_p * pl.elt / 16);
  p.gI = static_cast<const unsigned char*>(a.L);
  p.gI_end = p.gI + static_cast<size_t>(pl.s.i_n * pl.s.i_h * pl.s.i_w * pl.s.i_c) * pl.elt;
  p.k_h = static_cast<int>(pl.s.k_h);
  p.i_h = pl.s.i_h;
  p.i_w = pl.s.i_w;
  p.row_bytes = static_cast<int>(pl.s.i_w * pl.s.i_c * pl.elt);
  p.row_pitch = gather_row_pitch(pl);
  p.kwc = static_cast<int>(pl.s.k_w * pl.s.i_c);
  p.wstep_b = static_cast<int>(pl.s_w * pl.s.i_c * pl.elt);
  p.fused = a.fused;
  p.ncb = static_cast<int>(pl.s.i_c / pl.bk);
  p.k_w = static_cast<int>(pl.s.k_w);
  p.s_h = pl.s_h;
  p.s_w = pl.s_w;
  p.pad_h = pl.pad_h;
  p.pad_w = pl.pad_w;

  p.bn = pl.bn;
  p.n_tiles_n = pl.n_tiles_n;
  p.n_var = a.fused ? 1 : pl.n_var;  // the fused path uses weight variant 0 only
  p.avec = pl.avec;
  p.n_combo = p.n_var * pl.n_tiles_n;
  if (p.n_combo > kMaxCombos) return cudaErrorInvalidConfiguration;
  // first h of each weight variant: delta(h) = (h shift) mod vec = v delta_step
  for (int v = 0; v < 16; ++v) p.h_first[v] = static_cast<int>(pl.o_h);  // none
  if (a.fused) {
    p.h_first[0] = 0;
  } else {
    for (int64_t h = 0; h < std::min<int64_t>(pl.o_h, pl.n_var); ++h) {
      const int v = static_cast<int>(((h * pl.shift) % pl.avec) / pl.delta_step);
      if (p.h_first[v] > h) p.h_first[v] = static_cast<int>(h);
    }
  }
  p.out_hnwc = a.out_hnwc;
#ifdef MEC_TRACE
  if (const char* e = getenv("MEC_DEBUG_FLAGS")) p.dbg = atoi(e);
#endif
  p.spin = false;
  if (const char* e = getenv("MEC_GATHER_SPIN")) p.spin = gather && atoi(e) != 0;
  p.backoff_ns = 0;
  if (const char* e = getenv("MEC_GATHER_BACKOFF")) p.backoff_ns = gather ? static_cast<uint32_t>(atoi(e)) : 0u;
  if (const char* e = getenv("MEC_EPI_BACKOFF")) p.backoff_ns = gather ? p.backoff_ns : static_cast<uint32_t>(atoi(e));
  p.idesc = ptx::instr_desc(tf32, kBM, pl.bn);
  p.kchunk = 32 / pl.elt;
  p.kchunk_log2 = pl.elt == 2 ? 4 : 3;
  p.kdim = static_cast<int>(pl.kdim);
  p.n_chunks = static_cast<int>((pl.kdim + p.kchunk - 1) / p.kchunk);

  // epilogue: pass width = 128 / 64 / 32 bytes per row, dividing bn
  p.tma_store = ((pl.s.k_c * out_elt) % 16 == 0) && (reinterpret_cast<uintptr_t>(a.O) % 16 == 0);
  int row_bytes = 128;
  while (row_bytes > 32 && (pl.bn * out_elt) % row_bytes != 0) row_bytes /= 2;
  p.pw = row_bytes / out_elt;
  p.n_pass = pl.bn / p.pw;
  // a store box wider than the tensor's k_c extent traps (seen on B200 for
  // k_c = 8 with a 16-column box): such shapes use the register-store path
  if (pl.s.k_c % p.pw != 0) p.tma_store = false;
  p.stage_out_bytes = static_cast<uint32_t>(32 * row_bytes);  // 1-4 KB, swizzle-atom aligned
  p.epi_bufs = epi_bufs(gather);
  if (p.tma_store) {
    if (a.out_hnwc && flat) {  // O_hnwc viewed as {k_c, i_n o_w, o_h}
      const uint64_t dims[3] = {static_cast<uint64_t>(pl.s.k_c),
                                static_cast<uint64_t>(pl.s.i_n * pl.o_w),
                                static_cast<uint64_t>(pl.o_h)};
      const uint64_t strides[2] = {static_cast<uint64_t>(pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.s.i_n * pl.o_w * pl.s.k_c) * out_elt};
      const uint32_t box[3] = {static_cast<uint32_t>(p.pw), 32, 1};
      cudaError_t e = encode_tiled_swz(&tmO, tf32, 3, a.O, dims, strides, box, row_bytes);
      if (e != cudaSuccess) return e;
    } else if (a.out_hnwc) {  // O_hnwc viewed as {k_c, o_w, i_n, o_h}
      const uint64_t dims[4] = {static_cast<uint64_t>(pl.s.k_c), static_cast<uint64_t>(pl.o_w),
                                static_cast<uint64_t>(pl.s.i_n), static_cast<uint64_t>(pl.o_h)};
      const uint64_t strides[3] = {static_cast<uint64_t>(pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.o_w * pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.s.i_n * pl.o_w * pl.s.k_c) * out_elt};
      const uint32_t box[4] = {static_cast<uint32_t>(p.pw), 32, 1, 1};
      cudaError_t e = encode_tiled_swz(&tmO, tf32, 4, a.O, dims, strides, box, row_bytes);
      if (e != cudaSuccess) return e;
    } else {  // O viewed as {k_c, o_w, o_h, i_n}
      const uint64_t dims[4] = {static_cast<uint64_t>(pl.s.k_c), static_cast<uint64_t>(pl.o_w),
                                static_cast<uint64_t>(pl.o_h), static_cast<uint64_t>(pl.s.i_n)};
      const uint64_t strides[3] = {static_cast<uint64_t>(pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.o_w * pl.s.k_c) * out_elt,
                                   static_cast<uint64_t>(pl.o_h * pl.o_w * pl.s.k_c) * out_elt};
      const uint32_t box[4] = {static_cast<uint32_t>(p.pw), 32, 1, 1};
      cudaError_t e = encode_tiled_swz(&tmO, tf32, 4, a.O, dims, strides, box, row_bytes);
      if (e != cudaSuccess) return e;
    }
  } else {
    std::memset(&tmO, 0, sizeof(tmO));
  }

  const size_t b_tile = static_cast<size_t>(pl.bn) * kTileKBytes;
  const size_t b_res = b_tile * p.n_atoms;
  const size_t epi = epi_bytes(pl, gather);
  const size_t budget = kSmemBudget - epi;
  if (gather) p.slot_bytes = static_cast<uint32_t>(gather_slot_bytes(pl, ipt));
  if (gather) {
    // as many staged-row slots (2..4) as fit next to the resident weights: the
    // rows of tile t are requested when tile t - n_slots has been built
    const size_t fixed = b_res + p.n_atoms * 32 + 64;
    p.n_slots = 2;
    while (p.n_slots < 4 && fixed + (p.n_slots + 1) * static_cast<size_t>(p.slot_bytes) <= budget) ++p.n_slots;
  }
  const size_t gather_bytes =
      gather ? p.n_slots * static_cast<size_t>(p.slot_bytes) + p.n_atoms * 32 + 64 : 0;
  if (gather_bytes > budget) return cudaErrorInvalidConfiguration;
  const size_t budget_g = budget - gather_bytes;
  // gather: A atoms live in TMEM, so only the weights need shared memory
  p.resident = gather ? b_res <= budget_g
                      : (b_res + 2 * kMaxAtomsPerStage * kAtomBytes <= budget_g && b_res <= 120 * 1024);
  if (gather && !p.resident) return cudaErrorInvalidConfiguration;
  p.aps = (p.resident && !gather) ? 2 : 1;
  if (const char* e = getenv("MEC_APS"))  // (experiments) K-atoms per pipeline stage with resident weights
    if (p.resident && !gather) p.aps = std::max(1, std::min(6, atoi(e)));
  const size_t stage_a = gather ? 0 : static_cast<size_t>(p.aps) * kAtomBytes;
  p.n_kstages = (p.n_atoms + p.aps - 1) / p.aps;
  int stages;
  if (gather) {
    stages = 8;  // set from the TMEM budget below
  } else if (p.resident) {
    stages = static_cast<int>(std::min<size_t>(8, (budget_g - b_res) / stage_a));
  } else {
    stages = static_cast<int>(std::min<size_t>(8, budget_g / (stage_a + p.aps * b_tile)));
  }
  // multi-row tiles (see GemmParams::R)
  // Multi-row tiles (requested via mec_options_t::rows_per_tile) are parity-
  // tested, but with SS operands the extra B reads make them shared-memory-
  // bound on B200 (slower than R = 1), so auto = 1.
  // rows_per_tile 0 = auto: 4 (measured: C3 165 -> 142 us, C2 575 -> 500 us),
  // capped by TMEM (2 accumulator sets of R x bn columns)
  const int rpt = a.rows_per_tile > 0 ? a.rows_per_tile : (getenv("MEC_AUTO_R") ? atoi(getenv("MEC_AUTO_R")) : 4);
  p.R = 1;
  if (rpt > 1 && !a.fused && pl.n_var == 1 && p.resident && pl.shift % p.kchunk == 0 &&
      pl.shift < pl.kdim && pl.o_h > 1) {
    const int r = static_cast<int>(std::min<int64_t>({8, 512 / (2 * pl.bn), pl.o_h}));
    p.R = std::max(1, std::min(r, rpt));
  }
#ifdef MEC_TRACE
  if (const char* e = getenv("MEC_DEBUG_R")) {
    if (!a.fused && pl.n_var == 1 && p.resident && pl.shift % p.kchunk == 0 && pl.shift < pl.kdim && pl.o_h > 1)
      p.R = std::max(1, std::min<int>(std::min<int64_t>({8, 512 / (2 * pl.bn), pl.o_h}), atoi(e)));
  }
#endif
  p.shift_atoms = pl.shift % pl.bk == 0 ? static_cast<int>(pl.shift / pl.bk) : 0;
  p.shift_chunks = static_cast<int>(pl.shift / p.kchunk);
  p.n_acc = p.R > 1 ? 2 : (4 * pl.bn <= 512 ? 4 : 2);
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(p.n_acc * p.R * pl.bn)) cols <<= 1;
  p.tmem_cols = cols;
  if (gather) {
    // TMEM: n_acc accumulators, then A stages of 32 columns (128 bytes per row)
    // as many accumulators as leave >= 4 A stages (>= 2 for the widest N tiles)
    p.n_acc = 1;
    for (int k = 4; k >= 2; --k)
      if ((k * pl.bn + 31) / 32 * 32 + 4 * 32 <= 512) { p.n_acc = k; break; }
    if (const char* e = getenv("MEC_GATHER_NACC")) {
      const int k = atoi(e);
      if (k >= 1 && (k * pl.bn + 31) / 32 * 32 + 2 * 32 <= 512) p.n_acc = k;
    }
    p.a_col0 = static_cast<uint32_t>((p.n_acc * pl.bn + 31) / 32 * 32);
    p.tmem_cols = 512;
    stages = static_cast<int>(std::min<uint32_t>(8, (512 - p.a_col0) / 32));
    while (stages & (stages - 1)) --stages;  // a power of two (builders' stage arithmetic)
  }
  stages = std::max(1, std::min(stages, std::max(2, 2 * p.n_kstages)));
#ifdef MEC_TRACE
  if (const char* e = getenv("MEC_DEBUG_STAGES")) stages = std::min(stages, atoi(e));
#endif
  if (gather)
    while (stages & (stages - 1)) --stages;
  p.stages = stages;
  const size_t smem = kSmemAlign + stages * stage_a +
                      (p.resident ? b_res : stages * p.aps * b_tile) + epi + gather_bytes +
                      (2 * stages + 18) * 8 + 32;

  // grid: a multiple of the combo count, at most one CTA per SM
  int64_t max_tiles = 0;
  for (int v = 0; v < p.n_var; ++v) {
    const int64_t nh = p.R == 1 ? (pl.o_h - p.h_first[v] + p.n_var - 1) / p.n_var
                                : (pl.o_h + p.R - 1) / p.R;
    max_tiles = std::max<int64_t>(max_tiles, std::max<int64_t>(0, nh) * p.n_mt * groups);
  }
  if (max_tiles == 0) return cudaSuccess;
  int64_t per = std::max<int64_t>(1, num_sms() / p.n_combo);
  per = std::min<int64_t>(per, max_tiles);
  p.ctas_per_combo = static_cast<int>(per);
  p.tiles32 = max_tiles + per < (1LL << 31) && pl.o_h < (1LL << 31) && pl.s.i_n * pl.o_w < (1LL << 31);
  const int64_t grid = per * p.n_combo;
  auto kern = tf32 ? (gather ? window_gemm_kernel<true, true> : window_gemm_kernel<true, false>)
                   : (gather ? window_gemm_kernel<false, true> : window_gemm_kernel<false, false>);
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int threads = gather ? kernel_threads<true>() : kernel_threads<false>();
  // programmatic dependent launch: the kernel may start while the preceding
  // lowering / weight-prep kernel finishes (only the loads of its outputs wait)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = getenv("MEC_NO_PDL") ? 0 : 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmO, p);
  if (e != cudaSuccess) return e;
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace mec
