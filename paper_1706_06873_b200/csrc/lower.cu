// lower.cu -- MEC compact lowering on sm_100a (Alg.2 l.3-6):
//
//   L[n, w, h, 0:k_w, 0:i_c] = I[n, h, s_w w : s_w w + k_w, 0:i_c]
//
// for all n < i_n, w < o_w, h < i_h.  A pure bit copy; HBM-bound.
//
// B200 design: one CTA owns a band of HB input rows of one image.  It stages
// I[n, h0:h0+HB, :, :] (contiguous in NHWC) into shared memory
// with 128-bit coalesced loads -- every input byte is read from HBM once --
// then, for every output column w, writes the contiguous L segment
// L[n, w, h0:h0+HB, :, :] (HB strips of k_w i_c elements, adjacent in L)
// with 128-bit stores.  One warp per segment; a lane assembles one 16-byte
// output granule:
//   * aligned fast path (i_c elt a multiple of 16, e.g. i_c = 64 bf16):
//     one LDS.128 per STG.128;
//   * general path (e.g. i_c = 3): a granule inside one strip is a run of
//     contiguous smem elements at any alignment -> aligned 32-bit LDS +
//     funnel shifts; a granule straddling two strips falls back to element
//     loads.  All index math is 32-bit, one division per granule.
// HB is a multiple of 16/gcd(kwc elt,16) where possible so every segment of
// the pitch-padded conv-path L starts 16-byte aligned.
//
// The same launch also builds the GEMM's weight operand (Alg.2 l.7, "K as
// k_h k_w i_c x k_c matrix"), K-major and delta-shifted (see mec_internal.h),
// with 32x32 tiles transposed through shared memory by the CTAs after the
// lowering CTAs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <cstdio>
#include <cstdlib>

#include "mec_internal.h"
#include "ptx.cuh"

#ifdef MEC_TRACE
// Debug-only per-CTA timestamps of the lowering (separate libmec_trace.so,
// tools/trace_lower.py): [band][0] staged rows arrived, [1] copies built,
// [2] band written, [3] SM id
__device__ unsigned long long* g_lower_trace = nullptr;
extern "C" int mec_lower_trace_enable(void** dev_buf_out, size_t* bytes_out) {
  const size_t bytes = static_cast<size_t>(1 << 16) * 4 * 8;
  void* buf = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
  cudaMemset(buf, 0, bytes);
  if (cudaMemcpyToSymbol(g_lower_trace, &buf, sizeof(buf)) != cudaSuccess) return 2;
  *dev_buf_out = buf;
  *bytes_out = bytes;
  return 0;
}
__device__ __forceinline__ void lower_trace(int ev, long long idx) {
  unsigned long long* b = g_lower_trace;
  if (b != nullptr && threadIdx.x == 0 && idx < (1 << 16)) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    b[idx * 4 + ev] = t;
    if (ev == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      b[idx * 4 + 3] = smid;
    }
  }
}
#define LOWER_TRACE(ev) lower_trace(ev, b)
#else
#define LOWER_TRACE(ev) \
  do {                  \
  } while (0)
#endif

namespace mec {
namespace {

// host: a failed attribute / occupancy call is reported (MEC_DEBUG_ERRORS=1)
// and its error cleared, so it is not mistaken for a launch error later
inline cudaError_t host_ck(cudaError_t e, int line) {
  if (e != cudaSuccess) {
    if (getenv("MEC_DEBUG_ERRORS"))
      fprintf(stderr, "lower.cu:%d: %s\n", line, cudaGetErrorString(e));
    cudaGetLastError();
  }
  return e;
}
#define HOST_CK(x) host_ck((x), __LINE__)

struct LowerParams {
  const unsigned char* I;
  const unsigned char* I_end;
  unsigned char* L;
  int64_t i_h;
  int64_t pitch;  // L row pitch, elements
  int64_t o_w;
  uint32_t iwc;   // i_w i_c   (one input row, elements)
  uint32_t kwc;   // k_w i_c   (one strip, elements)
  uint32_t kwcs;  // strip stride in L (elements): kwc, or kwc padded with zeros (conv path, strip padding)
  uint32_t wstep; // s_w i_c   (strip start advance per output column)
  uint32_t kwc_magic;  // floor(2^32 / kwc) + 1: e / kwc == umulhi(e, magic) for e < 2^20
  int hb;         // input rows per CTA
  uint32_t table_off;  // smem byte offset of the word table (general path)
  int bands;      // ceil(i_h / hb)
  int64_t n_lower_blocks;
  // weight operand
  const unsigned char* K;
  unsigned char* Kt;
  int64_t kdim, k_c, kdim_pad, kc_pad;
  int n_var, delta_step;
  int64_t kwc_src, kwc_pad;  // gather layout: Kt column a kwc_pad + j <- K_mat row a kwc_src + j (0: identity)
  // zero padding (NEXT-4): i_h / iwc above are the padded extents; the caller's
  // I has src_h rows of src_iwc elements; staged rows are padded in smem
  bool padded;
  int64_t src_h, pad_h;
  uint32_t src_iwc, pad_wc;  // pad_wc = pad_w i_c elements
  bool aligned;   // fast path: every strip and segment 16-byte aligned
  // aligned-copies path (strips not 16-byte aligned, segments are; see
  // lower_copies): ncls staged copies of the band, copy k placed so that
  // every 16-byte output granule of the output columns of class k is one
  // aligned 16-byte shared-memory word
  int ncls;           // 0: path off
  int gcls_log2;      // log2 of g = gcd(delta16, wstep_b, 16); class value v = k g
  uint32_t copy_bytes;  // smem bytes per copy region
  uint32_t delta16;   // (i_w - k_w) i_c elt mod 16
  int wcls;           // column-class period 16 / gcd(wstep_b, 16)
  uint32_t raw_bytes;   // smem bytes per raw band buffer (two, double-buffered)
  int n_raw;            // raw band buffers: 2 (persistent CTAs, next band prefetched) or 1 (one band per CTA)
  int64_t total_bands;  // i_n bands (the persistent CTAs loop over them)
  bool prep_first;      // plain path: weight-prep CTAs before the lowering CTAs (large K)
  bool prep64;          // weight prep in 64 x 64 tiles with 16-byte vectors (bf16, k_c % 8 == 0)
  bool direct;          // aligned-copies path without the copies: every output granule is
                        // extracted from the raw band (two aligned LDS.128 per part)
  // words the next kernel needs zeroed (the wide window GEMM's split-K
  // counters), cleared by the last CTA of this launch
  uint32_t* zero_words;
  uint32_t n_zero;
  // row-copy path (lower_rows_kernel): 16-byte vectors per strip / per L row
  uint32_t vps, vpr, vps_magic;
  int64_t n_rows;          // i_n o_w rows of L
  int rows_per_cta;
};

template <typename T>
__device__ __forceinline__ void prep_weight_tile(const LowerParams& p, int64_t tile64) {
  // Kt[v][c][j] = K[j - v*delta_step][c] where 0 <= j - v*delta_step < kdim
  // and c < k_c; zero elsewhere.  32x32 tiles transposed through smem.
  // 32-bit index math (tile, row and column indices all fit) and four loads
  // in flight per thread before the smem stores: the 64-bit divisions and
  // one-load-at-a-time loop made this instruction- and latency-bound
  // (ncu, cv12 weight prep: 2600 warp instructions per tile, long-scoreboard
  // stalls dominant).
  __shared__ T tbuf[32][33];
  const uint32_t tiles_j = static_cast<uint32_t>((p.kdim_pad + 31) / 32);
  const uint32_t tiles_c = static_cast<uint32_t>((p.kc_pad + 31) / 32);
  uint32_t tile = static_cast<uint32_t>(tile64);
  const uint32_t v = tile / (tiles_j * tiles_c);
  tile -= v * tiles_j * tiles_c;
  const uint32_t jt = tile % tiles_j, ct = tile / tiles_j;
  const int32_t delta = static_cast<int32_t>(v * p.delta_step);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const T* K = reinterpret_cast<const T*>(p.K);
  T* Kt = reinterpret_cast<T*>(p.Kt) + static_cast<int64_t>(v) * p.kc_pad * p.kdim_pad;
  const int32_t kdim = static_cast<int32_t>(p.kdim), k_c = static_cast<int32_t>(p.k_c);
  const int32_t kwc_pad = static_cast<int32_t>(p.kwc_pad), kwc_src = static_cast<int32_t>(p.kwc_src);
  const int32_t c = static_cast<int32_t>(ct * 32 + tx);
  for (int r0 = ty; r0 < 32; r0 += 4 * nw) {
    T val[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = r0 + k * nw;
      int32_t j = static_cast<int32_t>(jt * 32) + r - delta;
      bool ok = r < 32 && j >= 0;
      if (kwc_pad > 0 && ok) {  // gather layout: per-kernel-row padding
        const int32_t a = j / kwc_pad, rr = j - a * kwc_pad;
        ok = rr < kwc_src;
        j = a * kwc_src + rr;
      }
      val[k] = (ok && j < kdim && c < k_c) ? K[static_cast<int64_t>(j) * k_c + c] : T(0);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (r0 + k * nw < 32) tbuf[r0 + k * nw][tx] = val[k];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += nw) {
    const int64_t cc = ct * 32 + r, jj = jt * 32 + tx;
    if (cc < p.kc_pad && jj < p.kdim_pad) Kt[cc * p.kdim_pad + jj] = tbuf[tx][r];
  }
  __syncthreads();
}

constexpr uint32_t kPrep64Stride = 66;  // elements per smem row (odd word count: 33)
constexpr size_t kPrep64Smem = 64 * kPrep64Stride * 2;

// The same Kt as prep_weight_tile, in 64 (j) x 64 (c) tiles of 2-byte elements:
// 16-byte loads along c (k_c % 8 == 0, so a vector is wholly in or out of
// range) into the launch's dynamic shared memory, then 16-byte stores along j
// (kdim_pad % 64 == 0), eight lanes per 128-byte row segment of Kt.
__device__ __forceinline__ void prep_weight_tile64(const LowerParams& p, uint32_t tile, unsigned char* sm) {
  uint16_t* tb = reinterpret_cast<uint16_t*>(sm);
  const uint32_t tiles_j = static_cast<uint32_t>(p.kdim_pad / 64);
  const uint32_t tiles_c = static_cast<uint32_t>((p.kc_pad + 63) / 64);
  const uint32_t v = tile / (tiles_j * tiles_c);
  tile -= v * tiles_j * tiles_c;
  const uint32_t jt = tile % tiles_j, ct = tile / tiles_j;
  const int32_t delta = static_cast<int32_t>(v * p.delta_step);
  const uint16_t* K = reinterpret_cast<const uint16_t*>(p.K);
  uint16_t* Kt = reinterpret_cast<uint16_t*>(p.Kt) + static_cast<int64_t>(v) * p.kc_pad * p.kdim_pad;
  const int32_t kdim = static_cast<int32_t>(p.kdim), k_c = static_cast<int32_t>(p.k_c);
  const int32_t kwc_pad = static_cast<int32_t>(p.kwc_pad), kwc_src = static_cast<int32_t>(p.kwc_src);
  for (uint32_t i = threadIdx.x; i < 512; i += blockDim.x) {
    const uint32_t r = i >> 3, cv = i & 7;
    int32_t j = static_cast<int32_t>(jt * 64 + r) - delta;
    const int32_t c = static_cast<int32_t>(ct * 64 + cv * 8);
    bool ok = j >= 0;
    if (kwc_pad > 0 && ok) {  // gather / strip-padded layout: per-kernel-row padding
      const int32_t a = j / kwc_pad, rr = j - a * kwc_pad;
      ok = rr < kwc_src;
      j = a * kwc_src + rr;
    }
    uint4 val = make_uint4(0, 0, 0, 0);
    if (ok && j < kdim && c < k_c) val = *reinterpret_cast<const uint4*>(K + static_cast<int64_t>(j) * k_c + c);
    uint32_t* d = reinterpret_cast<uint32_t*>(tb + r * kPrep64Stride + cv * 8);
    d[0] = val.x;
    d[1] = val.y;
    d[2] = val.z;
    d[3] = val.w;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 512; i += blockDim.x) {
    const uint32_t jv = i & 7, cr = i >> 3;
    const int64_t c = static_cast<int64_t>(ct) * 64 + cr;
    if (c < p.kc_pad) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = static_cast<uint32_t>(tb[(jv * 8 + 2 * q) * kPrep64Stride + cr]) |
               (static_cast<uint32_t>(tb[(jv * 8 + 2 * q + 1) * kPrep64Stride + cr]) << 16);
      *reinterpret_cast<uint4*>(Kt + c * p.kdim_pad + jt * 64 + jv * 8) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ int64_t prep_units(const LowerParams& p) {
  if (sizeof(T) == 2 && p.prep64) return p.n_var * (p.kdim_pad / 64) * ((p.kc_pad + 63) / 64);
  return p.n_var * ((p.kdim_pad + 31) / 32) * ((p.kc_pad + 31) / 32);
}

template <typename T>
__device__ __forceinline__ void prep_unit(const LowerParams& p, int64_t t, unsigned char* sm) {
  if (sizeof(T) == 2 && p.prep64)
    prep_weight_tile64(p, static_cast<uint32_t>(t), sm);
  else
    prep_weight_tile<T>(p, t);
}

// bytes [4 KK + sh_b / 8, + 16) of the 32-byte little-endian string x:y
template <int KK>
__device__ __forceinline__ uint4 extract16(uint4 x, uint4 y, uint32_t sh_b) {
  const uint32_t a[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
  return make_uint4(__funnelshift_r(a[KK], a[KK + 1], sh_b), __funnelshift_r(a[KK + 1], a[KK + 2], sh_b),
                    __funnelshift_r(a[KK + 2], a[KK + 3], sh_b), __funnelshift_r(a[KK + 3], a[KK + 4], sh_b));
}

// 16 bytes at byte offset o (0..15; k = o / 4, sh_b = 8 (o mod 4)) of the
// 32-byte little-endian string x:y, k and sh_b loop-invariant for the caller.
__device__ __forceinline__ uint4 extract16_rt(uint4 x, uint4 y, uint32_t k, uint32_t sh_b) {
  const uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
  uint32_t z[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) z[j] = k == 0 ? w[j] : (k == 1 ? w[j + 1] : (k == 2 ? w[j + 2] : w[j + 3]));
  return make_uint4(__funnelshift_r(z[0], z[1], sh_b), __funnelshift_r(z[1], z[2], sh_b),
                    __funnelshift_r(z[2], z[3], sh_b), __funnelshift_r(z[3], z[4], sh_b));
}

// Build one copy from the raw staged band: smem granule m (dst + 16 m) =
// raw bytes [r0 + 16 m, + 16), r0 = 16 KK' + sh_b / 8 relative to the
// 16-aligned raw address src (KK, sh_b uniform over the CTA).
template <int KK>
__device__ __forceinline__ void build_copy(uint32_t dst, uint32_t src, uint32_t sh_b, uint32_t n16) {
  for (uint32_t m = threadIdx.x; m < n16; m += blockDim.x) {
    const uint4 x = ptx::ld_shared_v4(src + 16 * m);
    const uint4 y = ptx::ld_shared_v4(src + 16 * m + 16);
    const uint4 v = extract16<KK>(x, y, sh_b);
    ptx::st_shared_v4(dst + 16 * m, v.x, v.y, v.z, v.w);
  }
}

// Aligned-copies lowering (strips of k_w i_c elements that are not 16-byte
// aligned, e.g. AlexNet conv1's 66-byte strips, into a segment-aligned L).
// Output granule q (16 bytes) of segment L[n, w, h0 : h0 + rows] holds bytes
// of strip hh = 16q / kwc_b (and, if it straddles, of strip hh + 1).  Strip
// hh of column w starts at band byte  hh iwc_b + w wstep_b  and at segment
// byte hh kwc_b, so source and destination differ by
//   v = hh (iwc_b - kwc_b) + w wstep_b  (mod 16), a multiple of g.
// Copy k = v / g of the band is staged at offset (16 - v) mod 16 inside its
// 16-aligned region: the granule is then one aligned LDS.128 (two, merged by
// a byte mask, when it straddles) and one STG.128 -- no per-byte shuffling in
// the output loop (the word-table path is instruction-bound on that).
//
// Persistent CTAs loop over the bands.  Band i + 1 is bulk-copied
// (cp.async.bulk, one DMA of the contiguous rows) into the other raw buffer
// while band i is built and written, so the HBM latency of the staging is
// hidden (a per-thread load loop serialised ~6 latencies per band: measured
// 5 us of a 15 us kernel for C1).
// Threads: granule q = tid mod nch, columns w = tid / nch + i wpar, with wpar
// a multiple of the column-class period 16 / gcd(wstep_b, 16), so a thread's
// copy never changes along its w loop (constant address increments).
template <typename T>
__device__ __forceinline__ void lower_copies(const LowerParams& p, unsigned char* smem, int64_t cta) {
  const uint32_t iwc_b = p.iwc * sizeof(T), kwc_b = p.kwc * sizeof(T);
  const uint32_t kwcs_b = p.kwcs * sizeof(T);  // strip stride in L (>= kwc_b; zero padded)
  const uint32_t wstep_b = p.wstep * sizeof(T);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  const uint32_t s_base = ptx::smem_u32(smem);
  const uint32_t raw0 = s_base + 128 + 32;  // raw buffer b at raw0 + b raw_bytes (32 B slack before)
  const uint32_t cps = s_base + 128 + static_cast<uint32_t>(p.n_raw) * p.raw_bytes;
  const int64_t nb = p.total_bands;
  const int64_t b0 = cta, bstep = p.n_lower_blocks;
#ifdef MEC_TRACE
  lower_trace(0, 32768 + cta);  // CTA entry (bank 2: per persistent CTA)
#endif
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // band -> (image, first row, rows, global start); issues its raw DMA
  auto band_src = [&](int64_t b, const unsigned char*& G, uint32_t& rows, int64_t& n, int64_t& h0) {
    n = b / p.bands;
    h0 = (b - n * p.bands) * static_cast<int64_t>(p.hb);
    rows = static_cast<uint32_t>(min(static_cast<int64_t>(p.hb), p.i_h - h0));
    G = p.I + static_cast<size_t>((n * p.i_h + h0) * p.iwc) * sizeof(T);
  };
  auto issue = [&](int64_t b, int buf) {
    const unsigned char* G;
    uint32_t rows;
    int64_t n, h0;
    band_src(b, G, rows, n, h0);
    const uintptr_t g = reinterpret_cast<uintptr_t>(G);
    const unsigned char* al = reinterpret_cast<const unsigned char*>(g & ~uintptr_t(15));
    const unsigned char* end = G + rows * iwc_b;
    const unsigned char* bulk_end =
        reinterpret_cast<const unsigned char*>(reinterpret_cast<uintptr_t>(end < p.I_end ? end + 15 : p.I_end) &
                                               ~uintptr_t(15));
    const uint32_t bytes = static_cast<uint32_t>(bulk_end - al);
    unsigned char* dst = smem + 128 + 32 + static_cast<size_t>(buf) * p.raw_bytes;
    // the very end of I may fall inside a 16-byte granule: its last bytes by plain loads
    for (const unsigned char* t = bulk_end; t < end; ++t) dst[t - al] = *t;
    ptx::mbar_arrive_expect_tx(&bars[buf], bytes);
    if (bytes > 0) ptx::bulk_load(dst, al, bytes, &bars[buf]);
  };
  if (threadIdx.x == 0 && b0 < nb) issue(b0, 0);

  // per-thread granule setup, cached per band height
  uint32_t set_rows = 0, wpar = 0, x0 = 0, off1 = 0, off2 = 0, m0 = 0, m1 = 0, m2 = 0, m3 = 0, n_it = 0;
  uint32_t n0 = 0, n1 = 0, n2 = 0, n3 = 0;
  uint32_t yb1 = 0, yb2 = 0;  // band bytes of granule byte 0 of parts 1 and 2 (direct mode)
  uint32_t wi = 0;
  bool idle = true;
  const uint32_t gsh = static_cast<uint32_t>(p.gcls_log2);
  int it = 0;
  for (int64_t b = b0; b < nb; b += bstep, ++it) {
    const int buf = it & 1;
    if (threadIdx.x == 0 && b + bstep < nb) issue(b + bstep, buf ^ 1);
    const unsigned char* G;
    uint32_t rows;
    int64_t n, h0;
    band_src(b, G, rows, n, h0);
    if (rows != set_rows) {
      set_rows = rows;
      const uint32_t nch = (rows * kwcs_b + 15) / 16;
      wpar = blockDim.x / nch;
      wpar -= wpar % static_cast<uint32_t>(p.wcls);  // >= wcls (host: nch(hb) wcls <= blockDim)
      const uint32_t q = threadIdx.x % nch;
      wi = threadIdx.x / nch;
      idle = wi >= wpar || wi >= static_cast<uint32_t>(p.o_w);
      x0 = 16 * q;
      const uint32_t hh = x0 / kwcs_b, r0 = x0 - hh * kwcs_b;
      // granule byte j: strip hh data for j < cut1, zero padding for
      // cut1 <= j < cut2, strip hh + 1 data for j >= cut2 (kwcs_b >= 16: no
      // granule reaches strip hh + 2)
      const uint32_t cut1 = r0 >= kwc_b ? 0u : min(16u, kwc_b - r0);
      const uint32_t cut2 = hh + 1 >= rows ? 16u : min(16u, kwcs_b - r0);
      auto range_mask = [](uint32_t lo, uint32_t hi, uint32_t b0) -> uint32_t {  // bytes [lo, hi) of word b0..b0+3
        uint32_t m = 0;
        for (uint32_t b = 0; b < 4; ++b)
          if (b0 + b >= lo && b0 + b < hi) m |= 0xFFu << (8 * b);
        return m;
      };
      m0 = range_mask(0, cut1, 0);
      m1 = range_mask(0, cut1, 4);
      m2 = range_mask(0, cut1, 8);
      m3 = range_mask(0, cut1, 12);
      n0 = range_mask(cut2, 16, 0);
      n1 = range_mask(cut2, 16, 4);
      n2 = range_mask(cut2, 16, 8);
      n3 = range_mask(cut2, 16, 12);
      // band byte y of copy k sits at cps + k copy_bytes + 16 + o_k + y
      const uint32_t y1 = hh * iwc_b + r0 + wi * wstep_b;  // part 1: band byte of granule byte 0
      const uint32_t v1 = (hh * p.delta16 + wi * wstep_b) & 15u;
      off1 = (v1 >> gsh) * p.copy_bytes + 16u + ((16u - v1) & 15u) + y1;
      off2 = off1;  // part 2 (strip hh + 1), = part 1 if unused
      yb1 = y1;
      yb2 = cut2 < 16 ? y1 + iwc_b - kwcs_b : y1;
      if (cut2 < 16) {
        const uint32_t y2 = y1 + iwc_b - kwcs_b;
        const uint32_t v2 = (v1 + p.delta16) & 15u;
        off2 = (v2 >> gsh) * p.copy_bytes + 16u + ((16u - v2) & 15u) + y2;
      }
      n_it = idle ? 0u : (static_cast<uint32_t>(p.o_w) - wi + wpar - 1) / wpar;
    }
    ptx::mbar_wait(&bars[buf], static_cast<uint32_t>(it >> 1) & 1u);
    LOWER_TRACE(0);
    // ---- build the copies: copy k granule m = band bytes [16 m - 16 - o_k, + 16) ----
    const uint32_t band_b = rows * iwc_b;
    const uint32_t n16 = (band_b + 31) / 16 + 2;
    const uint32_t g15 = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(G) & 15);
    const uint32_t rawb = raw0 + static_cast<uint32_t>(buf) * p.raw_bytes;  // band byte y at rawb + g15 + y
    if (p.direct) {
      // ---- output straight from the raw band: granule part 1 (and 2) are the
      // 16 bytes at raw address a (a mod 16 fixed along the w loop: da is a
      // multiple of 16), taken out of the two aligned 16-byte words around it ----
      uint32_t a1 = rawb + g15 + yb1, a2 = rawb + g15 + yb2;
      const uint32_t k1 = (a1 >> 2) & 3u, s1 = (a1 & 3u) * 8u, k2 = (a2 >> 2) & 3u, s2 = (a2 & 3u) * 8u;
      a1 &= ~15u;
      a2 &= ~15u;
      const uint32_t da = wpar * wstep_b;
      const size_t pitch_b = static_cast<size_t>(p.pitch) * sizeof(T);
      unsigned char* dst = p.L + ((n * p.o_w + wi) * p.pitch + h0 * p.kwcs) * sizeof(T) + x0;
      const size_t dstep = pitch_b * wpar;
#pragma unroll 2
      for (uint32_t i = 0; i < n_it; ++i) {
        const uint4 x = extract16_rt(ptx::ld_shared_v4(a1), ptx::ld_shared_v4(a1 + 16), k1, s1);
        const uint4 y = extract16_rt(ptx::ld_shared_v4(a2), ptx::ld_shared_v4(a2 + 16), k2, s2);
        uint4 o;
        o.x = (x.x & m0) | (y.x & n0);
        o.y = (x.y & m1) | (y.y & n1);
        o.z = (x.z & m2) | (y.z & n2);
        o.w = (x.w & m3) | (y.w & n3);
        *reinterpret_cast<uint4*>(dst) = o;
        a1 += da;
        a2 += da;
        dst += dstep;
      }
      __syncthreads();  // this raw buffer is rewritten next
      LOWER_TRACE(2);
      continue;
    }
    for (int k = 0; k < p.ncls; ++k) {
      const uint32_t o_k = (16u - (static_cast<uint32_t>(k) << gsh)) & 15u;
      const uint32_t r = rawb + g15 - 16u - o_k;  // raw address of copy granule 0 (>= raw0 - 32)
      const uint32_t src = r & ~15u, sh = r & 15u, sh_b = (sh & 3u) * 8u;
      const uint32_t dst = cps + static_cast<uint32_t>(k) * p.copy_bytes;
      switch (sh >> 2) {
        case 0: build_copy<0>(dst, src, sh_b, n16); break;
        case 1: build_copy<1>(dst, src, sh_b, n16); break;
        case 2: build_copy<2>(dst, src, sh_b, n16); break;
        default: build_copy<3>(dst, src, sh_b, n16); break;
      }
    }
    __syncthreads();
    LOWER_TRACE(1);
    // ---- output ----
    uint32_t a1 = cps + off1, a2 = cps + off2;
    const uint32_t da = wpar * wstep_b;  // a multiple of 16: same copy every iteration
    const size_t pitch_b = static_cast<size_t>(p.pitch) * sizeof(T);
    unsigned char* dst = p.L + ((n * p.o_w + wi) * p.pitch + h0 * p.kwcs) * sizeof(T) + x0;
    const size_t dstep = pitch_b * wpar;
#pragma unroll 4
    for (uint32_t i = 0; i < n_it; ++i) {
      const uint4 x = ptx::ld_shared_v4(a1);
      const uint4 y = ptx::ld_shared_v4(a2);
      uint4 o;
      o.x = (x.x & m0) | (y.x & n0);
      o.y = (x.y & m1) | (y.y & n1);
      o.z = (x.z & m2) | (y.z & n2);
      o.w = (x.w & m3) | (y.w & n3);
      *reinterpret_cast<uint4*>(dst) = o;
      a1 += da;
      a2 += da;
      dst += dstep;
    }
    __syncthreads();  // the copies and this raw buffer are rewritten next
    LOWER_TRACE(2);
  }
#ifdef MEC_TRACE
  lower_trace(2, 32768 + cta);  // CTA exit
#endif
}

template <typename T>
__global__ void __launch_bounds__(512) lower_kernel(const LowerParams p) {
  constexpr uint32_t VEC = 16 / sizeof(T);
  extern __shared__ __align__(16) unsigned char smem[];
  // the window GEMM that follows is launched as a programmatic dependent: let
  // its prologue start now (its loads of L / Kt wait for this grid to finish)
  ptx::griddep_launch_dependents();
  if (p.zero_words != nullptr && blockIdx.x == gridDim.x - 1)
    for (uint32_t i = threadIdx.x; i < p.n_zero; i += blockDim.x) p.zero_words[i] = 0u;

  if (p.ncls > 0) {
    // persistent lowering CTAs after the weight-prep CTAs, which are thus
    // scheduled first instead of waiting for a free slot at the end
    const int64_t n_prep = gridDim.x - p.n_lower_blocks;
    if (blockIdx.x < n_prep) {
      const int64_t n_tiles = prep_units<T>(p);
      for (int64_t t = blockIdx.x; t < n_tiles; t += n_prep) prep_unit<T>(p, t, smem);
      return;
    }
    lower_copies<T>(p, smem, static_cast<int64_t>(blockIdx.x) - n_prep);
    return;
  }
  // weight-prep CTAs: after the lowering CTAs (they fill the tail), or first
  // when K is large (cv12 / cv6, MBs of K: placed last they ran their tile
  // loops as a serial tail, measured)
  const int64_t n_prep = gridDim.x - p.n_lower_blocks;
  const int64_t prep_idx = p.prep_first ? static_cast<int64_t>(blockIdx.x)
                                        : static_cast<int64_t>(blockIdx.x) - p.n_lower_blocks;
  if (prep_idx >= 0 && prep_idx < n_prep) {
    const int64_t n_tiles = prep_units<T>(p);
    for (int64_t t = prep_idx; t < n_tiles; t += n_prep) prep_unit<T>(p, t, smem);
    return;
  }

  const int64_t blk = static_cast<int64_t>(blockIdx.x) - (p.prep_first ? n_prep : 0);
  const int64_t n = blk / p.bands;
  const int64_t h0 = (blk % p.bands) * static_cast<int64_t>(p.hb);
  const uint32_t rows = static_cast<uint32_t>(min(static_cast<int64_t>(p.hb), p.i_h - h0));

  uint32_t shift_elems = 0;
  if (p.padded) {
    // ---- stage rows h0..h0+rows of the zero-padded image: zero the band,
    // then copy the source rows it covers at column offset pad_w i_c ----
    const uint32_t nz = (rows * p.iwc * static_cast<uint32_t>(sizeof(T)) + 15) / 16 + 3;
    for (uint32_t i = threadIdx.x; i < nz; i += blockDim.x)
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    for (uint32_t hh = 0; hh < rows; ++hh) {
      const int64_t y = h0 + hh - p.pad_h;
      if (y < 0 || y >= p.src_h) continue;
      const T* src = reinterpret_cast<const T*>(p.I) + (n * p.src_h + y) * p.src_iwc;
      T* dst = reinterpret_cast<T*>(smem) + hh * p.iwc + p.pad_wc;
      const uint32_t row_b = p.src_iwc * static_cast<uint32_t>(sizeof(T));
      if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (row_b & 15) == 0) {
        // 128-bit loads; stores at the padded (possibly 2-byte aligned) offset
        const uint4* s16 = reinterpret_cast<const uint4*>(src);
        unsigned char* db = reinterpret_cast<unsigned char*>(dst);
        const bool w4 = (reinterpret_cast<uintptr_t>(db) & 3) == 0;
        for (uint32_t i = threadIdx.x; i < row_b / 16; i += blockDim.x) {
          const uint4 v = __ldg(s16 + i);
          unsigned char* d = db + 16 * i;
          if (w4) {
            uint32_t* d4 = reinterpret_cast<uint32_t*>(d);
            d4[0] = v.x;
            d4[1] = v.y;
            d4[2] = v.z;
            d4[3] = v.w;
          } else {
            uint16_t* d2 = reinterpret_cast<uint16_t*>(d);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              d2[2 * k] = static_cast<uint16_t>(w[k] & 0xFFFFu);
              d2[2 * k + 1] = static_cast<uint16_t>(w[k] >> 16);
            }
          }
        }
      } else {
        for (uint32_t e = threadIdx.x; e < p.src_iwc; e += blockDim.x) dst[e] = src[e];
      }
    }
    __syncthreads();
  } else {
  // ---- stage I[n, h0:h0+rows, :, :] in shared memory (128-bit loads) ----
  const unsigned char* a0 = p.I + ((n * p.i_h + h0) * p.iwc) * sizeof(T);
  const unsigned char* ab = reinterpret_cast<const unsigned char*>(
      reinterpret_cast<uintptr_t>(a0) & ~static_cast<uintptr_t>(15));
  shift_elems = static_cast<uint32_t>((a0 - ab) / sizeof(T));
  const uint32_t nbytes = static_cast<uint32_t>(a0 - ab) + rows * p.iwc * sizeof(T);
  const uint32_t n16 = (nbytes + 15) / 16;
  for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) {
    const unsigned char* g = ab + 16 * static_cast<size_t>(i);
    if (g + 16 <= p.I_end) {
      *reinterpret_cast<uint4*>(smem + 16 * i) = __ldg(reinterpret_cast<const uint4*>(g));
    } else {
      for (uint32_t b = 0; b < VEC; ++b) {
        const unsigned char* ge = g + b * sizeof(T);
        if (ge < p.I_end)
          reinterpret_cast<T*>(smem + 16 * i)[b] = *reinterpret_cast<const T*>(ge);
      }
    }
  }
  // zero the slack past the staged bytes so table reads past a row end are defined
  if (threadIdx.x < 3) reinterpret_cast<uint4*>(smem + 16 * n16)[threadIdx.x] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  }

  const T* srow = reinterpret_cast<const T*>(smem) + shift_elems;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  (void)warp;
  (void)lane;
  (void)nwarps;
  const uint32_t seg_len = rows * p.kwc;  // elements of L[n, w, h0:h0+rows, :, :]

  if (p.aligned) {
    // every strip starts 16-byte aligned in both smem and L: 1 LDS.128 per STG.128;
    // (w, vector) flattened over the CTA
    const uint32_t vps = p.kwc / VEC;  // vectors per strip
    const uint32_t n_vec = rows * vps;
    const uint32_t total = n_vec * static_cast<uint32_t>(p.o_w);
    for (uint32_t idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const uint32_t w = idx / n_vec, v = idx - w * n_vec;
      const uint32_t hh = v / vps, r = (v - hh * vps) * VEC;
      T* dst = reinterpret_cast<T*>(p.L) + (n * p.o_w + w) * p.pitch + h0 * p.kwc;
      *reinterpret_cast<uint4*>(dst + hh * p.kwc + r) =
          *reinterpret_cast<const uint4*>(srow + w * p.wstep + hh * p.iwc + r);
    }
    return;
  }

  // general path (strips not 16-byte aligned, e.g. i_c = 3).  When every
  // segment starts 4-byte aligned (pitch-padded conv-path L), each 4-byte
  // output word j of a segment is byte_perm(W[a_j], W[b_j], sel_j) of two
  // aligned 32-bit words of the staged rows, with (a_j, b_j, sel_j) the same
  // for every w up to the word shift w*wstep*elt/4 (two tables: that shift's
  // 2-byte remainder).  Per word: table LDS + 2 LDS + PRMT + STG, consecutive
  // lanes on consecutive words (conflict-free, coalesced).
  const uint32_t seg_bytes = seg_len * sizeof(T);
  const bool word_ok = (p.pitch * sizeof(T)) % 4 == 0 &&
                       ((reinterpret_cast<uintptr_t>(p.L) + h0 * p.kwc * sizeof(T)) & 3) == 0;
  if (word_ok) {
    const uint32_t seg_words = (seg_bytes + 3) / 4;
    uint32_t* table = reinterpret_cast<uint32_t*>(smem + p.table_off);
    const uint32_t sbyte0 = shift_elems * sizeof(T);
    for (uint32_t t = threadIdx.x; t < 2 * seg_words; t += blockDim.x) {
      const uint32_t par = t / seg_words, j = t - par * seg_words;
      uint32_t wa, wb, sel;
      if constexpr (sizeof(T) == 4) {
        const uint32_t hh = p.kwc_magic ? __umulhi(j, p.kwc_magic) : j;
        const uint32_t r = j - hh * p.kwc;
        wa = (sbyte0 + (hh * p.iwc + r) * 4) >> 2;
        wb = wa;
        sel = 0;  // 0x3210
      } else {
        const uint32_t e0 = 2 * j, e1 = 2 * j + 1 < seg_len ? 2 * j + 1 : 2 * j;
        const uint32_t h0e = p.kwc_magic ? __umulhi(e0, p.kwc_magic) : e0;
        const uint32_t h1e = p.kwc_magic ? __umulhi(e1, p.kwc_magic) : e1;
        const uint32_t b0 = sbyte0 + (h0e * p.iwc + e0 - h0e * p.kwc) * 2 + par * 2;
        const uint32_t b1 = sbyte0 + (h1e * p.iwc + e1 - h1e * p.kwc) * 2 + par * 2;
        wa = b0 >> 2;
        wb = b1 >> 2;
        sel = ((b0 >> 1) & 1u) | (((b1 >> 1) & 1u) << 1);
      }
      table[t] = wa | (wb << 15) | (sel << 30);
    }
    __syncthreads();
    const uint32_t* W = reinterpret_cast<const uint32_t*>(smem);
    const bool odd_tail = (seg_bytes & 3u) != 0;  // last word holds one 2-byte element
    unsigned char* L0 = p.L + (((n * p.o_w) * p.pitch + h0 * p.kwc) * sizeof(T));
    const uint32_t pitch_bytes = static_cast<uint32_t>(p.pitch * sizeof(T));
    const uint32_t wstep_bytes = p.wstep * static_cast<uint32_t>(sizeof(T));
    // one warp per 32-word column block, looping over every output column w:
    // the lane's table entries are decoded once; the inner loop is 2 LDS +
    // PRMT + STG with incremental addresses (the launch sizes the block to
    // the number of column blocks)
    const uint32_t nblk = (seg_words + 31) / 32;
    const uint32_t full_words = odd_tail ? seg_words - 1 : seg_words;
    // warps beyond the column blocks split the w loop: warp = jb + nblk * wpart
    const uint32_t wsplit = nwarps >= nblk ? nwarps / nblk : 1u;
    const uint32_t wpart = warp / nblk;
    if (wpart >= wsplit) return;
    for (uint32_t jb = warp - wpart * nblk; jb < nblk; jb += (wsplit == 1 ? nwarps : nblk * 1000000u)) {
      const uint32_t j = jb * 32 + lane;
      const bool active = j < full_words;
      const uint32_t jj = j < seg_words ? j : seg_words - 1;
      const uint32_t e0 = table[jj], e1 = table[seg_words + jj];
      const uint32_t a0 = e0 & 0x7FFFu, b0 = (e0 >> 15) & 0x7FFFu;
      const uint32_t a1 = e1 & 0x7FFFu, b1 = (e1 >> 15) & 0x7FFFu;
      const uint32_t s0 = ((e0 >> 30) & 1u ? 0x0032u : 0x0010u) | ((e0 >> 31) ? 0x7600u : 0x5400u);
      const uint32_t s1 = ((e1 >> 30) & 1u ? 0x0032u : 0x0010u) | ((e1 >> 31) ? 0x7600u : 0x5400u);
      // this warp's columns w = wpart, wpart + wsplit, ...
      uint32_t wbyte = wpart * wstep_bytes;
      uint32_t* dst = reinterpret_cast<uint32_t*>(L0 + 4 * jj + static_cast<size_t>(wpart) * pitch_bytes);
      const uint32_t dst_step = pitch_bytes * wsplit;
      const uint32_t wb_step = wstep_bytes * wsplit;
      if (active && (wstep_bytes & 3u) == 0) {
        // word-aligned column step (e.g. AlexNet conv1: 24 B): parity 0 always
        const uint32_t wstep_words = (wstep_bytes >> 2) * wsplit;
        const uint32_t* xa = W + a0 + (wbyte >> 2);
        const uint32_t* xb = W + b0 + (wbyte >> 2);
        const uint32_t n_w = static_cast<uint32_t>(p.o_w);
#pragma unroll 4
        for (uint32_t w = wpart; w < n_w; w += wsplit) {
          const uint32_t x = *xa;
          uint32_t val = x;
          if constexpr (sizeof(T) == 2) val = __byte_perm(x, *xb, s0);
          *dst = val;
          xa += wstep_words;
          xb += wstep_words;
          dst = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(dst) + dst_step);
        }
      } else if (active) {
        for (uint32_t w = wpart; w < static_cast<uint32_t>(p.o_w); w += wsplit) {
          const bool par = (wbyte >> 1) & 1u;
          const uint32_t* Wb = W + (wbyte >> 2);
          const uint32_t x = Wb[par ? a1 : a0];
          uint32_t val = x;
          if constexpr (sizeof(T) == 2) val = __byte_perm(x, Wb[par ? b1 : b0], par ? s1 : s0);
          *dst = val;
          wbyte += wb_step;
          dst = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(dst) + dst_step);
        }
      } else if (odd_tail && j == seg_words - 1) {  // the segment's last 2-byte element
        for (uint32_t w = wpart; w < static_cast<uint32_t>(p.o_w); w += wsplit) {
          const bool par = (wbyte >> 1) & 1u;
          const uint32_t x = W[(wbyte >> 2) + (par ? a1 : a0)];
          const uint32_t lo = ((par ? e1 : e0) >> 30) & 1u ? (x >> 16) : (x & 0xFFFFu);
          *reinterpret_cast<uint16_t*>(dst) = static_cast<uint16_t>(lo);
          wbyte += wb_step;
          dst = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(dst) + dst_step);
        }
      }
    }
    return;
  }

  // non-uniform segment alignment (dense L with an odd pitch, mec_lower):
  // element-wise, one warp per segment
  for (uint32_t w = warp; w < p.o_w; w += nwarps) {
    T* seg = reinterpret_cast<T*>(p.L) + (n * p.o_w + w) * p.pitch + h0 * p.kwc;
    for (uint32_t e = lane; e < seg_len; e += 32) {
      const uint32_t h2 = p.kwc_magic ? __umulhi(e, p.kwc_magic) : e;
      const uint32_t r2 = e - h2 * p.kwc;
      seg[e] = srow[h2 * p.iwc + w * p.wstep + r2];
    }
  }
}

// Direct fallback for input rows too wide to stage in shared memory: every
// thread copies one L element from global.  (Not used by any BASELINE config.)
// Row-copy lowering for strips that are whole 16-byte vectors (i_c elt a
// multiple of 16: C2, C3, cv4-cv12).  Alg.2 l.4-6: L[n,w,h,:,:] = I[n,h,s_w
// w : s_w w + k_w,:] -- every strip is one contiguous run of k_w i_c elements
// of I, so each 16-byte vector of L is one 16-byte vector of I: a CTA copies
// whole rows (n, w) of L (i_h strips) straight from global to global, a warp
// reading and writing 512 contiguous bytes per instruction.  No shared
// memory, no barrier: many independent loads in flight per SM (the staged
// band kernel waited for its band before writing).  The k_w / s_w-fold
// re-reads of I (neighbouring w share pixels) are served by L2.  Zero
// padding (NEXT-4): vectors of pixels outside the unpadded image are zeros.
// Blocks past the L rows prepare the weight operand (as lower_kernel).
#ifndef MEC_ROWS_UNROLL
#define MEC_ROWS_UNROLL 4  // 16-byte vectors in flight per thread (row-copy lowering)
#endif
template <typename T>
__global__ void __launch_bounds__(256) lower_rows_kernel(const LowerParams p) {
  constexpr uint32_t VEC = 16 / sizeof(T);
  extern __shared__ __align__(16) unsigned char smem[];
  ptx::griddep_launch_dependents();
  if (p.zero_words != nullptr && blockIdx.x == gridDim.x - 1)
    for (uint32_t i = threadIdx.x; i < p.n_zero; i += blockDim.x) p.zero_words[i] = 0u;
  const int64_t row_blocks = (p.n_rows + p.rows_per_cta - 1) / p.rows_per_cta;
  if (static_cast<int64_t>(blockIdx.x) >= row_blocks) {
    const int64_t n_prep = gridDim.x - row_blocks;
    const int64_t n_tiles = prep_units<T>(p);
    for (int64_t t = blockIdx.x - row_blocks; t < n_tiles; t += n_prep) prep_unit<T>(p, t, smem);
    return;
  }
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * p.rows_per_cta;
  const int64_t r1 = min(p.n_rows, r0 + p.rows_per_cta);
  const uint4* I4 = reinterpret_cast<const uint4*>(p.I);
  for (int64_t row = r0; row < r1; ++row) {
    const int64_t n = row / p.o_w, w = row - n * p.o_w;
    uint4* dst = reinterpret_cast<uint4*>(p.L + static_cast<size_t>(row * p.pitch) * sizeof(T));
    // vector u of the row: strip h = u / vps, vector j = u mod vps of the strip
    for (uint32_t u0 = threadIdx.x; u0 < p.vpr; u0 += MEC_ROWS_UNROLL * blockDim.x) {
      uint4 v[MEC_ROWS_UNROLL];
#pragma unroll
      for (int k = 0; k < MEC_ROWS_UNROLL; ++k) {
        const uint32_t u = u0 + k * blockDim.x;
        v[k] = make_uint4(0u, 0u, 0u, 0u);
        if (u < p.vpr) {
          // (vps == 1: the magic number 2^32 + 1 does not fit; h = u)
          const uint32_t h = p.vps == 1 ? u : __umulhi(u, p.vps_magic), j = u - h * p.vps;
          if (!p.padded) {
            const int64_t e = ((n * p.i_h + h) * p.iwc + static_cast<int64_t>(w) * p.wstep) / VEC + j;
            v[k] = __ldg(I4 + e);
          } else {
            // padded image: row h - pad_h, element column w s_w i_c + j VEC - pad_w i_c
            const int64_t y = static_cast<int64_t>(h) - p.pad_h;
            const int64_t xc = static_cast<int64_t>(w) * p.wstep + static_cast<int64_t>(j) * VEC - p.pad_wc;
            if (y >= 0 && y < p.src_h && xc >= 0 && xc < p.src_iwc)
              v[k] = __ldg(I4 + ((n * p.src_h + y) * p.src_iwc + xc) / VEC);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < MEC_ROWS_UNROLL; ++k) {
        const uint32_t u = u0 + k * blockDim.x;
        if (u < p.vpr) dst[u] = v[k];
      }
    }
  }
}

// Row-gather lowering for strips that are not whole 16-byte vectors (i_c = 3:
// AlexNet conv1 / cv1-cv3, cv7).  Each thread writes one 16-byte vector of an
// L row (n, w): its VEC elements e come from strip h = e / (k_w i_c), element
// j = e mod (k_w i_c), i.e. I[n, h, s_w w + j / i_c, j mod i_c] (Alg.2 l.4-6) --
// consecutive within a strip, a vector spanning at most two strips.  Element
// loads (a warp's loads fall in a few contiguous runs of I: L1/L2 hits for the
// k_w / s_w-fold re-reads), one 16-byte store.  Rows past l_cols in the
// pitched L (pitch padding) are written with whatever the clamped gather
// reads (never read by a GEMM: the weight rows there are zero).
template <typename T>
__global__ void __launch_bounds__(256) lower_rows_gather_kernel(const LowerParams p) {
  constexpr uint32_t VEC = 16 / sizeof(T);
  extern __shared__ __align__(16) unsigned char smem[];
  ptx::griddep_launch_dependents();
  if (p.zero_words != nullptr && blockIdx.x == gridDim.x - 1)
    for (uint32_t i = threadIdx.x; i < p.n_zero; i += blockDim.x) p.zero_words[i] = 0u;
  const int64_t row_blocks = (p.n_rows + p.rows_per_cta - 1) / p.rows_per_cta;
  if (static_cast<int64_t>(blockIdx.x) >= row_blocks) {
    const int64_t n_prep = gridDim.x - row_blocks;
    const int64_t n_tiles = prep_units<T>(p);
    for (int64_t t = blockIdx.x - row_blocks; t < n_tiles; t += n_prep) prep_unit<T>(p, t, smem);
    return;
  }
  const T* Ie = reinterpret_cast<const T*>(p.I);
  const uint32_t lcols = static_cast<uint32_t>(p.i_h) * p.kwc;  // valid elements of an L row
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * p.rows_per_cta;
  const int64_t r1 = min(p.n_rows, r0 + p.rows_per_cta);
  for (int64_t row = r0; row < r1; ++row) {
    const int64_t n = row / p.o_w, w = row - n * p.o_w;
    T* dst = reinterpret_cast<T*>(p.L) + static_cast<size_t>(row * p.pitch);
    const T* src_row = Ie + n * p.i_h * p.iwc + static_cast<int64_t>(w) * p.wstep;  // strip h at + h iwc
    for (uint32_t u = threadIdx.x; u < p.vpr; u += blockDim.x) {
      uint32_t e = u * VEC;
      // first element's strip and offset (magic division by kwc, exact for e < 2^20)
      uint32_t h = __umulhi(e, p.kwc_magic), j = e - h * p.kwc;
      if (p.kwc == 1) { h = e; j = 0; }
      T val[VEC];
#pragma unroll
      for (uint32_t k = 0; k < VEC; ++k) {
        if (e + k < lcols) {
          val[k] = __ldg(src_row + static_cast<int64_t>(h) * p.iwc + j);
        } else {
          val[k] = T(0);
        }
        if (++j == p.kwc) {
          j = 0;
          ++h;
        }
      }
      uint4 o;
      if constexpr (sizeof(T) == 2) {
        o.x = static_cast<uint32_t>(val[0]) | (static_cast<uint32_t>(val[1]) << 16);
        o.y = static_cast<uint32_t>(val[2]) | (static_cast<uint32_t>(val[3]) << 16);
        o.z = static_cast<uint32_t>(val[4]) | (static_cast<uint32_t>(val[5]) << 16);
        o.w = static_cast<uint32_t>(val[6]) | (static_cast<uint32_t>(val[7]) << 16);
      } else {
        o = make_uint4(val[0], val[1], val[2], val[3]);
      }
      reinterpret_cast<uint4*>(dst)[u] = o;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) lower_direct_kernel(const T* __restrict__ I, T* __restrict__ L,
                                                           int64_t i_n, int64_t i_h, int64_t i_w,
                                                           int64_t i_c, int64_t k_w, int64_t s_w,
                                                           int64_t o_w, int64_t pitch, int64_t src_h,
                                                           int64_t src_w, int64_t pad_h, int64_t pad_w,
                                                           int64_t kwcs) {
  // i_h / i_w: padded extents; I has src_h x src_w pixels (zero outside);
  // strips of k_w i_c elements at a stride of kwcs (>= k_w i_c, zero filled)
  const int64_t kwc = k_w * i_c, row = i_h * kwcs;
  const int64_t total = i_n * o_w * row;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t nw = e / row, rem = e - nw * row;
    const int64_t n = nw / o_w, w = nw - n * o_w;
    const int64_t h = rem / kwcs, r = rem - h * kwcs;
    const int64_t y = h - pad_h, x = s_w * w + r / i_c - pad_w;
    L[nw * pitch + rem] = (r < kwc && y >= 0 && y < src_h && x >= 0 && x < src_w)
                              ? I[((n * src_h + y) * src_w + x) * i_c + r % i_c]
                              : T(0);
  }
}

}  // namespace

// Kernel attributes, set once per process: the largest dynamic shared memory
// any lowering launch uses (setting it per call to that call's size would
// LOWER it for the next, larger launch -- a launch failure seen in the tests),
// and an all-shared carveout (the copies path sizes its grid to the resident
// CTAs; with the default L1-leaning carveout C1's bands took 2.25 waves).
constexpr size_t kLowerMaxSmem = 200 * 1024;
void set_lower_attributes() {
  // function attributes are per device: once per device, thread-safe
  static std::once_flag once[kMaxDevices];
  std::call_once(once[current_device()], [] {
    HOST_CK(cudaFuncSetAttribute(lower_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kLowerMaxSmem)));
    HOST_CK(cudaFuncSetAttribute(lower_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kLowerMaxSmem)));
    HOST_CK(cudaFuncSetAttribute(lower_kernel<uint16_t>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared));
    HOST_CK(cudaFuncSetAttribute(lower_kernel<uint32_t>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared));
  });
}

cudaError_t launch_lower(const Plan& pl, const void* I, void* L, int64_t pitch, const void* K,
                         void* Kt, cudaStream_t st, int* launches, bool gather_kt, uint32_t* zero_words,
                         uint32_t n_zero) {
  const mec_shape_t& s = pl.s;
  LowerParams p{};
  p.zero_words = n_zero > 0 ? zero_words : nullptr;
  p.n_zero = n_zero;
  p.I = static_cast<const unsigned char*>(I);
  p.I_end = p.I + static_cast<size_t>(s.i_n * pl.src_h * pl.src_w * s.i_c) * pl.elt;
  p.padded = pl.pad_h > 0 || pl.pad_w > 0;
  p.src_h = pl.src_h;
  p.pad_h = pl.pad_h;
  p.src_iwc = static_cast<uint32_t>(pl.src_w * s.i_c);
  p.pad_wc = static_cast<uint32_t>(pl.pad_w * s.i_c);
  p.L = static_cast<unsigned char*>(L);
  p.i_h = s.i_h;
  p.o_w = pl.o_w;
  p.pitch = pitch;
  p.iwc = static_cast<uint32_t>(s.i_w * s.i_c);
  p.kwc = static_cast<uint32_t>(s.k_w * s.i_c);
  p.kwcs = static_cast<uint32_t>(pl.strip);
  const bool spad = p.kwcs != p.kwc;  // strip-padded conv-path L (Plan::kwc_s)
  p.wstep = static_cast<uint32_t>(pl.s_w * s.i_c);
  p.kwc_magic = p.kwc > 1 ? static_cast<uint32_t>((1ull << 32) / p.kwc + 1) : 0u;  // 0: kwc == 1
  p.K = static_cast<const unsigned char*>(K);
  p.Kt = static_cast<unsigned char*>(Kt);
  p.kdim = pl.kdim;
  p.k_c = s.k_c;
  p.kdim_pad = pl.kdim_pad;
  p.kc_pad = pl.kc_pad;
  p.n_var = pl.n_var;
  p.delta_step = pl.delta_step;
  if (gather_kt) {
    p.n_var = 1;
    p.kdim_pad = pl.kdim_g;
    p.kwc_src = s.k_w * s.i_c;
    p.kwc_pad = pl.kwc_p;
  } else if (spad) {
    // strip-padded L: Kt column a kwc_s + j <- K_mat row a k_w i_c + j (same
    // layout as the gather path's operand), zero in the pad columns
    p.kdim = pl.kdim_src;
    p.kwc_src = s.k_w * s.i_c;
    p.kwc_pad = pl.kwc_s;
  }

  int64_t prep_blocks = 0;
  if (Kt != nullptr) {
    const int64_t tiles = p.n_var * ((p.kdim_pad + 31) / 32) * ((pl.kc_pad + 31) / 32);
    // (a 32 x 32 tile per loop trip).  Measured (DESIGN.md "Weight-prep
    // CTAs"): with >= 1024 tiles (cv12 2304, cv6 1152) the prep is the
    // critical path: those CTAs go first, about 4 tiles each (~4 resp. 2 per
    // SM).  Below (cv5 / cv11 ~600 tiles, C1 36) they go last, 2 per SM at
    // most, and fill the lowering's tail.
    p.prep_first = tiles >= 1024;
    // 64 x 64 tiles (one per prep CTA when they go first) where the vectors fit
    p.prep64 = pl.elt == 2 && s.k_c % 8 == 0 && p.kdim_pad % 64 == 0 &&
               reinterpret_cast<uintptr_t>(K) % 16 == 0 && reinterpret_cast<uintptr_t>(Kt) % 16 == 0 &&
               !getenv("MEC_PREP32");
    if (const char* e = getenv("MEC_PREP_FIRST")) p.prep_first = atoi(e) != 0;  // (experiments)
    const int64_t units = p.prep64 ? p.n_var * (p.kdim_pad / 64) * ((pl.kc_pad + 63) / 64) : tiles;
    const int64_t per_sm = getenv("MEC_PREP_PER_SM") ? atoi(getenv("MEC_PREP_PER_SM")) : 0;
    prep_blocks = std::min<int64_t>(units, per_sm > 0      ? per_sm * num_sms()
                                           : p.prep_first ? (p.prep64 ? units : (units + 3) / 4)
                                                          : 2LL * num_sms());
  }
  const size_t prep_smem = p.prep64 ? kPrep64Smem : 64;
  if (L == nullptr) {  // weight operand only (fused path)
    if (prep_blocks == 0) {
      if (p.zero_words != nullptr) return cudaMemsetAsync(p.zero_words, 0, p.n_zero * sizeof(uint32_t), st);
      return cudaSuccess;
    }
    LowerParams q = p;
    q.n_lower_blocks = 0;
    if (pl.elt == 2)
      lower_kernel<uint16_t><<<static_cast<unsigned>(prep_blocks), 256, prep_smem, st>>>(q);
    else
      lower_kernel<uint32_t><<<static_cast<unsigned>(prep_blocks), 256, prep_smem, st>>>(q);
    if (launches) ++*launches;
    return cudaGetLastError();
  }

  // Row-copy path (lower_rows_kernel): every strip a whole number of 16-byte
  // vectors at 16-byte aligned addresses on both sides (MEC_LOWER_ROWS=0: the
  // staged band kernel below)
  {
    const uint32_t vecn = static_cast<uint32_t>(16 / pl.elt);
    const bool rows_ok = !spad && p.kwc % vecn == 0 && p.wstep % vecn == 0 && p.iwc % vecn == 0 &&
                         pitch % vecn == 0 && (!p.padded || (p.src_iwc % vecn == 0 && p.pad_wc % vecn == 0)) &&
                         reinterpret_cast<uintptr_t>(I) % 16 == 0 && reinterpret_cast<uintptr_t>(L) % 16 == 0 &&
                         s.i_h * (p.kwc / vecn) < (1LL << 31) && s.i_n * pl.o_w < (1LL << 40) &&
                         // the magic-number division u / vps is exact for u vps < 2^32
                         static_cast<uint64_t>(s.i_h) * (p.kwc / vecn) * (p.kwc / vecn) < (1ull << 32);
    const char* er = getenv("MEC_LOWER_ROWS");
    if (rows_ok && (er == nullptr || atoi(er) != 0)) {
      LowerParams q = p;
      q.vps = p.kwc / vecn;
      q.vpr = static_cast<uint32_t>(s.i_h) * q.vps;
      q.vps_magic = static_cast<uint32_t>((1ull << 32) / q.vps + 1);
      q.n_rows = s.i_n * pl.o_w;
      // rows per CTA: ~8 vectors per thread (one unrolled trip of 4 x 256 x 2)
      q.rows_per_cta = static_cast<int>(std::max<int64_t>(1, 2048 / q.vpr));
      if (const char* e = getenv("MEC_LOWER_ROWS_PER_CTA")) q.rows_per_cta = std::max(1, atoi(e));
      const int64_t row_blocks = (q.n_rows + q.rows_per_cta - 1) / q.rows_per_cta;
      const int64_t grid = row_blocks + prep_blocks;
      if (grid > 0x7FFFFFFF) return cudaErrorInvalidConfiguration;
      const size_t rsmem = (q.prep64 && prep_blocks > 0) ? kPrep64Smem : 64;
      if (pl.elt == 2)
        lower_rows_kernel<uint16_t><<<static_cast<unsigned>(grid), 256, rsmem, st>>>(q);
      else
        lower_rows_kernel<uint32_t><<<static_cast<unsigned>(grid), 256, rsmem, st>>>(q);
      if (launches) ++*launches;
      return cudaGetLastError();
    }
  }
  // Row-gather path (lower_rows_gather_kernel) for the other unpadded layouts
  // with 16-byte aligned L rows.  Opt-in (MEC_LOWER_GATHER=1): measured slower
  // than the staged aligned-copies kernel below (AlexNet conv1 b32 22.9 vs
  // 15.9 us, cv3 b128 85 vs 55 us) -- one element load per 2-4 bytes of L.
  {
    const uint32_t vecn = static_cast<uint32_t>(16 / pl.elt);
    const char* eg = getenv("MEC_LOWER_GATHER");
    const bool g_ok = !spad && !p.padded && pitch % vecn == 0 && reinterpret_cast<uintptr_t>(L) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(I) % sizeof(uint16_t) == 0 && pl.l_cols < (1LL << 20) &&
                      s.i_n * pl.o_w < (1LL << 40);
    if (g_ok && eg != nullptr && atoi(eg) != 0) {
      LowerParams q = p;
      q.vpr = static_cast<uint32_t>((pl.l_cols + vecn - 1) / vecn);  // vectors covering l_cols (<= pitch)
      q.n_rows = s.i_n * pl.o_w;
      q.rows_per_cta = static_cast<int>(std::max<int64_t>(1, 1024 / q.vpr));
      if (const char* e = getenv("MEC_LOWER_ROWS_PER_CTA")) q.rows_per_cta = std::max(1, atoi(e));
      const int64_t row_blocks = (q.n_rows + q.rows_per_cta - 1) / q.rows_per_cta;
      const int64_t grid = row_blocks + prep_blocks;
      if (grid > 0x7FFFFFFF) return cudaErrorInvalidConfiguration;
      const size_t rsmem = (q.prep64 && prep_blocks > 0) ? kPrep64Smem : 64;
      if (pl.elt == 2)
        lower_rows_gather_kernel<uint16_t><<<static_cast<unsigned>(grid), 256, rsmem, st>>>(q);
      else
        lower_rows_gather_kernel<uint32_t><<<static_cast<unsigned>(grid), 256, rsmem, st>>>(q);
      if (launches) ++*launches;
      return cudaGetLastError();
    }
  }
  const int64_t row_bytes = static_cast<int64_t>(p.iwc) * pl.elt;
  const int64_t max_smem = 96 * 1024;
  bool use_smem = row_bytes + 64 <= max_smem && s.k_w * s.i_c < (1 << 20) && p.iwc < (1u << 24);
  // (the strip-padded layout is written by the aligned-copies path only, else
  // by the direct kernel: see below, after the band height is known)
  auto launch_direct = [&]() -> cudaError_t {
    // weight prep still needs the main kernel's prep blocks: run them with a 1-band grid
    if (Kt == nullptr && p.zero_words != nullptr) {
      const cudaError_t ez = cudaMemsetAsync(p.zero_words, 0, p.n_zero * sizeof(uint32_t), st);
      if (ez != cudaSuccess) return ez;
    }
    if (Kt != nullptr) {
      LowerParams q = p;
      q.n_lower_blocks = 0;
      if (pl.elt == 2)
        lower_kernel<uint16_t><<<static_cast<unsigned>(prep_blocks), 256, prep_smem, st>>>(q);
      else
        lower_kernel<uint32_t><<<static_cast<unsigned>(prep_blocks), 256, prep_smem, st>>>(q);
      if (launches) ++*launches;
    }
    const int64_t total = s.i_n * pl.o_w * pl.l_cols;
    const int64_t grid = std::min<int64_t>((total + 255) / 256, 32LL * num_sms());
    if (pl.elt == 2)
      lower_direct_kernel<uint16_t><<<static_cast<unsigned>(grid), 256, 0, st>>>(
          static_cast<const uint16_t*>(I), static_cast<uint16_t*>(L), s.i_n, s.i_h, s.i_w, s.i_c,
          s.k_w, pl.s_w, pl.o_w, pitch, pl.src_h, pl.src_w, pl.pad_h, pl.pad_w, p.kwcs);
    else
      lower_direct_kernel<uint32_t><<<static_cast<unsigned>(grid), 256, 0, st>>>(
          static_cast<const uint32_t*>(I), static_cast<uint32_t*>(L), s.i_n, s.i_h, s.i_w, s.i_c,
          s.k_w, pl.s_w, pl.o_w, pitch, pl.src_h, pl.src_w, pl.pad_h, pl.pad_w, p.kwcs);
    if (launches) ++*launches;
    return cudaGetLastError();
  };
  if (!use_smem) return launch_direct();

  // Rows per CTA: stage <= ~24 KB of input (several CTAs per SM), enough CTAs
  // for >= ~4 per SM, and HB a multiple of the alignment period so segments of
  // a 16-byte-pitched L start 16-byte aligned.
  const int vec = 16 / pl.elt;
  int64_t period = 1;
  while ((period * p.kwcs) % vec != 0) ++period;  // <= vec
  const int64_t max_rows_smem = std::max<int64_t>(1, (24 * 1024) / row_bytes);
  const int64_t want_blocks = 4LL * num_sms();
  int64_t hb = std::min<int64_t>(s.i_h, max_rows_smem);
  while (hb > period && s.i_n * ((s.i_h + hb - 1) / hb) < want_blocks) hb = (hb + 1) / 2;
  if (hb > period && hb < s.i_h) hb = hb / period * period;
  // the general path divides e < hb*kwc by kwc with a 32-bit magic multiply,
  // exact while hb*kwc*kwc < 2^32
  while (hb > 1 && static_cast<uint64_t>(hb) * p.kwc * p.kwc >= (1ull << 32)) hb = (hb + 1) / 2;
  hb = std::max<int64_t>(1, hb);
  if (const char* e = getenv("MEC_LOWER_HB"))  // (experiments: rows per band, a multiple of the period)
    hb = std::max<int64_t>(period, std::min<int64_t>(s.i_h, atoi(e) / period * period));
  p.hb = static_cast<int>(hb);
  p.bands = static_cast<int>((s.i_h + hb - 1) / hb);
  p.n_lower_blocks = s.i_n * p.bands;

  const bool base_ok = (reinterpret_cast<uintptr_t>(I) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(L) % 16 == 0);
  p.aligned = !spad && base_ok && (p.kwc % vec == 0) && (p.wstep % vec == 0) && (p.iwc % vec == 0) &&
              (pitch % vec == 0);

  // general (word-table) path: one warp per 32-word column block of a segment
  int threads = 256;
  if (!p.aligned) {
    // one warp per 32-word column block of a segment (up to 8), times wsplit
    // warp groups that split the w loop (more warps per staged band)
    const int64_t words = (hb * static_cast<int64_t>(p.kwc) * pl.elt + 3) / 4;
    const int64_t nblk = (words + 31) / 32;
    // (measured on B200 for AlexNet conv1: splitting the w loop over more warps
    // per band is slower -- 18.6 vs 16.5 us -- so 1 unless overridden)
    int64_t wsplit = 1;
    if (const char* e = getenv("MEC_LOWER_WSPLIT")) wsplit = std::max(1, atoi(e));
    if (nblk > 8) threads = 256;
    else threads = static_cast<int>(32 * std::max<int64_t>(2, std::min<int64_t>(16, nblk * wsplit)));
  }
  const size_t staged = static_cast<size_t>(hb * row_bytes) + 96;
  p.table_off = static_cast<uint32_t>((staged + 15) / 16 * 16);
  const size_t seg_words = (static_cast<size_t>(hb) * p.kwc * pl.elt + 3) / 4;
  size_t smem = p.table_off + (p.aligned ? 0 : 2 * seg_words * 4);

  // aligned-copies path (see lower_copies): strips of >= 16 bytes that are not
  // 16-byte aligned, 16-byte-aligned segments (pitch-padded L), few classes
  p.ncls = 0;
  if (!p.aligned && !p.padded && base_ok && !getenv("MEC_LOWER_NO_COPIES")) {
    const uint32_t kwc_b = p.kwcs * pl.elt, iwc_b = p.iwc * pl.elt, ws_b = p.wstep * pl.elt;  // (strip stride)
    const uint32_t seg_b = static_cast<uint32_t>(hb) * kwc_b;
    const bool seg_aligned = (pitch * pl.elt) % 16 == 0 && seg_b % 16 == 0;
    const uint32_t d16 = (iwc_b - kwc_b) & 15u;
    uint32_t g = 16;
    for (uint32_t x : {d16, ws_b & 15u}) {
      uint32_t a = g, b = x;
      while (b) { const uint32_t t = a % b; a = b; b = t; }
      g = a;
    }
    const int ncls = static_cast<int>(16 / g);
    const uint32_t n16 = (static_cast<uint32_t>(hb) * iwc_b + 31) / 16 + 2;
    const size_t csmem = static_cast<size_t>(ncls) * 16 * n16;
    const uint32_t nch = (seg_b + 15) / 16;
    uint32_t gw = 16, bw = ws_b & 15u;
    while (bw) { const uint32_t t = gw % bw; gw = bw; bw = t; }
    const uint32_t wcls = 16 / gw;
    const size_t raw_b = (32 + static_cast<size_t>(hb) * iwc_b + 128 + 15) / 16 * 16;
    if (kwc_b >= 16 && seg_aligned && ncls <= (spad ? 8 : 4) && 128 + 2 * raw_b + csmem <= kLowerMaxSmem &&
        nch * wcls <= 512) {
      p.ncls = ncls;
      int lg = 0;
      while ((1u << lg) < g) ++lg;
      p.gcls_log2 = lg;
      p.copy_bytes = 16 * n16;
      p.delta16 = d16;
      p.wcls = static_cast<int>(wcls);
      // columns per granule: a multiple of wcls; the block size with the fewest
      // idle lanes (ties: the larger block)
      uint32_t best_t = 0;
      double best_eff = -1.0;
      // (<= 256 threads: every thread then loops over several columns, which
      // amortises its per-granule setup -- measured: 480-thread blocks with 4
      // columns per thread spent most instructions in setup)
      // (measured: 256 for AlexNet conv1, o_w = 55 -- 16.0 us vs 18.0 at 384;
      // 512 for cv3 b128, o_w = 111 -- 54.9 vs 63.1 us)
      const uint32_t max_t = getenv("MEC_LOWER_MAXT") ? static_cast<uint32_t>(atoi(getenv("MEC_LOWER_MAXT")))
                                                      : (pl.o_w >= 100 ? 512u : 256u);
      for (uint32_t wp = wcls; nch * wp <= max_t || wp == wcls; wp += wcls) {
        const uint32_t t = (nch * wp + 31) / 32 * 32;
        const double eff = static_cast<double>(nch * wp) / t;
        if (eff >= best_eff - 1e-9) { best_eff = eff; best_t = t; }
        if (wp >= static_cast<uint32_t>(pl.o_w)) break;
      }
      threads = static_cast<int>(std::max<uint32_t>(best_t, 64));
      p.raw_bytes = static_cast<uint32_t>(raw_b);
      // direct extraction without the copies: opt-in (MEC_LOWER_DIRECT=1),
      // measured slower on B200 -- AlexNet conv1 22.4 vs 16.5 us, cv3 b128
      // 114 vs 63 us: the output loop is instruction-bound, not store-bound
      p.direct = getenv("MEC_LOWER_DIRECT") && atoi(getenv("MEC_LOWER_DIRECT")) != 0;
      p.total_bands = p.n_lower_blocks;
      // one band per CTA: one raw buffer, more CTAs per SM, the block scheduler
      // balances (measured on B200: cv1 b128 39.5 -> 36.4 us, cv3 b128 54.7 ->
      // 51.0, AlexNet conv1 unchanged); MEC_LOWER_ONE_BAND=0: persistent CTAs
      // with a prefetched second band (round 1)
      const bool one_band = !(getenv("MEC_LOWER_ONE_BAND") && atoi(getenv("MEC_LOWER_ONE_BAND")) == 0);
      p.n_raw = one_band ? 1 : 2;
      smem = 128 + static_cast<size_t>(p.n_raw) * p.raw_bytes + (p.direct ? 0 : csmem);
      // persistent CTAs: as many as are co-resident (each loops over bands,
      // prefetching the next band's rows while it writes the current one)
      int occ = 0;
      set_lower_attributes();
      if (pl.elt == 2)
        HOST_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lower_kernel<uint16_t>, threads, smem));
      else
        HOST_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lower_kernel<uint32_t>, threads, smem));
      occ = std::max(1, occ);
      if (const char* e = getenv("MEC_LOWER_CTAS_PER_SM")) occ = std::max(1, std::min(occ, atoi(e)));
      // equal band counts per CTA (a ragged last round of bands left most CTAs
      // idle while a quarter of them processed a second band: measured)
      const int64_t slots = static_cast<int64_t>(occ) * num_sms();
      const int64_t per = one_band ? 1 : (p.total_bands + slots - 1) / slots;
      p.n_lower_blocks = (p.total_bands + per - 1) / per;
    }
  }
  const int64_t grid = p.n_lower_blocks + prep_blocks;
  if (grid > 0x7FFFFFFF) return cudaErrorInvalidConfiguration;
  if (spad && p.ncls == 0) return launch_direct();
  set_lower_attributes();
  if (p.prep64 && prep_blocks > 0) smem = std::max(smem, kPrep64Smem);
  if (smem > kLowerMaxSmem) return cudaErrorInvalidConfiguration;
  if (pl.elt == 2)
    lower_kernel<uint16_t><<<static_cast<unsigned>(grid), threads, smem, st>>>(p);
  else
    lower_kernel<uint32_t><<<static_cast<unsigned>(grid), threads, smem, st>>>(p);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace mec
