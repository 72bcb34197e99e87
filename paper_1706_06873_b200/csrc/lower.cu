// lower.cu -- MEC compact lowering on sm_100a (Alg.2 l.3-6):
//
//   L[n, w, h, 0:k_w, 0:i_c] = I[n, h, s_w w : s_w w + k_w, 0:i_c]
//
// for all n < i_n, w < o_w, h < i_h.  A pure bit copy; HBM-bound.
//
// B200 design: one CTA owns a band of HB input rows of one image.  It stages
// I[n, h0:h0+HB, :, :] (contiguous in NHWC) into shared memory
// with 128-bit coalesced loads -- every input byte is read from HBM once --
// and then, for every output column w, writes the contiguous L segment
// L[n, w, h0:h0+HB, :, :] (HB strips of k_w i_c elements, which are
// adjacent in L) with 128-bit coalesced stores, gathering the strips
// from shared memory.  Segments that do not start 16-byte aligned get a
// scalar head/tail.  When every strip offset is 16-byte aligned (i_c elt a
// multiple of 16, e.g. i_c = 64 bf16) the gather is one 128-bit LDS per
// store.
//
// The same launch also builds the GEMM's weight operand (Alg.2 l.7, "K as
// k_h k_w i_c x k_c matrix"): Kt = K_mat^T, k_c_pad x kdim_pad, zero padded,
// K-major for tcgen05 -- 32x32 tiles transposed through shared memory by the
// CTAs after the lowering CTAs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mec_internal.h"

namespace mec {
namespace {

struct LowerParams {
  const unsigned char* I;
  const unsigned char* I_end;
  unsigned char* L;
  int64_t i_h, i_w, i_c, k_w, s_w, o_w;
  int64_t iwc;    // i_w i_c   (one input row, elements)
  int64_t kwc;    // k_w i_c   (one strip, elements)
  int64_t pitch;  // L row pitch, elements
  int hb;         // input rows per CTA
  int bands;      // ceil(i_h / hb)
  int64_t n_lower_blocks;
  // weight operand
  const unsigned char* K;
  unsigned char* Kt;
  int64_t kdim, k_c, kdim_pad, kc_pad;
  int n_var, delta_step;
  bool aligned;   // fast path: every strip and segment 16-byte aligned
};

template <typename T>
__device__ __forceinline__ void prep_weight_tile(const LowerParams& p, int64_t tile) {
  // Kt[v][c][j] = K[j - v*delta_step][c] where 0 <= j - v*delta_step < kdim
  // and c < k_c; zero elsewhere.  32x32 tiles transposed through smem.
  __shared__ T tbuf[32][33];
  const int64_t tiles_j = (p.kdim_pad + 31) / 32;
  const int64_t tiles_c = (p.kc_pad + 31) / 32;
  const int64_t v = tile / (tiles_j * tiles_c);
  tile -= v * tiles_j * tiles_c;
  const int64_t jt = tile % tiles_j, ct = tile / tiles_j;
  const int64_t delta = v * p.delta_step;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
  const T* K = reinterpret_cast<const T*>(p.K);
  T* Kt = reinterpret_cast<T*>(p.Kt) + v * p.kc_pad * p.kdim_pad;
  for (int r = ty; r < 32; r += 8) {
    const int64_t j = jt * 32 + r - delta, c = ct * 32 + tx;
    tbuf[r][tx] = (j >= 0 && j < p.kdim && c < p.k_c) ? K[j * p.k_c + c] : T(0);
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t c = ct * 32 + r, j = jt * 32 + tx;
    if (c < p.kc_pad && j < p.kdim_pad) Kt[c * p.kdim_pad + j] = tbuf[tx][r];
  }
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(256) lower_kernel(const LowerParams p) {
  constexpr int VEC = 16 / sizeof(T);
  extern __shared__ __align__(16) unsigned char smem[];

  if (blockIdx.x >= p.n_lower_blocks) {
    const int64_t n_tiles = p.n_var * ((p.kdim_pad + 31) / 32) * ((p.kc_pad + 31) / 32);
    for (int64_t t = blockIdx.x - p.n_lower_blocks; t < n_tiles;
         t += gridDim.x - p.n_lower_blocks)
      prep_weight_tile<T>(p, t);
    return;
  }

  const int64_t n = blockIdx.x / p.bands;
  const int64_t h0 = (blockIdx.x % p.bands) * p.hb;
  const int64_t rows = min(static_cast<int64_t>(p.hb), p.i_h - h0);

  // ---- stage I[n, h0:h0+rows, :, :] in shared memory (128-bit loads) ----
  const unsigned char* a0 = p.I + ((n * p.i_h + h0) * p.iwc) * sizeof(T);
  const unsigned char* ab = reinterpret_cast<const unsigned char*>(
      reinterpret_cast<uintptr_t>(a0) & ~static_cast<uintptr_t>(15));
  const int shift_elems = static_cast<int>((a0 - ab) / sizeof(T));
  const int64_t nbytes = (a0 - ab) + rows * p.iwc * sizeof(T);
  const int64_t n16 = (nbytes + 15) / 16;
  for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) {
    const unsigned char* g = ab + 16 * i;
    if (g + 16 <= p.I_end) {
      *reinterpret_cast<uint4*>(smem + 16 * i) = __ldg(reinterpret_cast<const uint4*>(g));
    } else {
      for (int b = 0; b < VEC; ++b) {
        const unsigned char* ge = g + b * sizeof(T);
        if (ge < p.I_end)
          reinterpret_cast<T*>(smem + 16 * i)[b] = *reinterpret_cast<const T*>(ge);
      }
    }
  }
  __syncthreads();

  const T* srow = reinterpret_cast<const T*>(smem) + shift_elems;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int64_t seg_len = rows * p.kwc;  // elements of L[n, w, h0:h0+rows, :, :]

  if (p.aligned) {
    // every strip starts 16-byte aligned in both smem and L: 1 LDS.128 per STG.128
    const int64_t vec_per_strip = p.kwc / VEC;
    const int64_t n_vec = rows * vec_per_strip;
    for (int64_t w = warp; w < p.o_w; w += nwarps) {
      T* dst = reinterpret_cast<T*>(p.L) + (n * p.o_w + w) * p.pitch + h0 * p.kwc;
      const T* src = srow + p.s_w * w * p.i_c;
      for (int64_t v = lane; v < n_vec; v += 32) {
        const int64_t hh = v / vec_per_strip, r = (v - hh * vec_per_strip) * VEC;
        const uint4 val = *reinterpret_cast<const uint4*>(src + hh * p.iwc + r);
        *reinterpret_cast<uint4*>(dst + hh * p.kwc + r) = val;
      }
    }
    return;
  }

  // general path: 16-byte granules of each L segment, gathered element-wise
  for (int64_t w = warp; w < p.o_w; w += nwarps) {
    T* seg = reinterpret_cast<T*>(p.L) + (n * p.o_w + w) * p.pitch + h0 * p.kwc;
    const T* src = srow + p.s_w * w * p.i_c;
    const int head = static_cast<int>((reinterpret_cast<uintptr_t>(seg) & 15) / sizeof(T));
    T* gbase = seg - head;  // 16-byte aligned
    const int64_t n_gran = (head + seg_len + VEC - 1) / VEC;
    for (int64_t gi = lane; gi < n_gran; gi += 32) {
      const int64_t e0 = gi * VEC - head;  // segment element of the granule's first slot
      int64_t hh = (e0 >= 0) ? e0 / p.kwc : 0;
      int64_t r = (e0 >= 0) ? e0 - hh * p.kwc : 0;
      if (e0 >= 0 && e0 + VEC <= seg_len) {
        union {
          uint4 v;
          T e[VEC];
        } u;
#pragma unroll
        for (int b = 0; b < VEC; ++b) {
          u.e[b] = src[hh * p.iwc + r];
          if (++r == p.kwc) { r = 0; ++hh; }
        }
        *reinterpret_cast<uint4*>(gbase + gi * VEC) = u.v;
      } else {
        for (int b = 0; b < VEC; ++b) {
          const int64_t e = e0 + b;
          if (e < 0 || e >= seg_len) continue;
          const int64_t h2 = e / p.kwc, r2 = e - h2 * p.kwc;
          gbase[gi * VEC + b] = src[h2 * p.iwc + r2];
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_lower(const Plan& pl, const void* I, void* L, int64_t pitch, const void* K,
                         void* Kt, cudaStream_t st, int* launches) {
  const mec_shape_t& s = pl.s;
  LowerParams p{};
  p.I = static_cast<const unsigned char*>(I);
  p.I_end = p.I + static_cast<size_t>(s.i_n * s.i_h * s.i_w * s.i_c) * pl.elt;
  p.L = static_cast<unsigned char*>(L);
  p.i_h = s.i_h;
  p.i_w = s.i_w;
  p.i_c = s.i_c;
  p.k_w = s.k_w;
  p.s_w = pl.s_w;
  p.o_w = pl.o_w;
  p.iwc = s.i_w * s.i_c;
  p.kwc = s.k_w * s.i_c;
  p.pitch = pitch;
  p.K = static_cast<const unsigned char*>(K);
  p.Kt = static_cast<unsigned char*>(Kt);
  p.kdim = pl.kdim;
  p.k_c = s.k_c;
  p.kdim_pad = pl.kdim_pad;
  p.kc_pad = pl.kc_pad;
  p.n_var = pl.n_var;
  p.delta_step = pl.delta_step;

  // Rows per CTA: stage at most ~24 KB of input and aim for >= ~4 CTAs per SM.
  const int64_t row_bytes = p.iwc * pl.elt;
  const int64_t max_rows_smem = std::max<int64_t>(1, (24 * 1024) / row_bytes);
  const int64_t want_blocks = 4LL * num_sms();
  int64_t hb = std::min<int64_t>(s.i_h, max_rows_smem);
  while (hb > 1 && s.i_n * ((s.i_h + hb - 1) / hb) < want_blocks) hb = (hb + 1) / 2;
  // keep each band's L segment 16-byte aligned where the strip length allows it
  p.hb = static_cast<int>(hb);
  p.bands = static_cast<int>((s.i_h + hb - 1) / hb);
  p.n_lower_blocks = s.i_n * p.bands;

  const int vec = 16 / pl.elt;
  const bool base_ok = (reinterpret_cast<uintptr_t>(I) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(L) % 16 == 0);
  p.aligned = base_ok && (p.kwc % vec == 0) && ((pl.s_w * s.i_c) % vec == 0) &&
              (p.iwc % vec == 0) && (pitch % vec == 0);

  const size_t smem = static_cast<size_t>(hb * row_bytes) + 32;
  int64_t prep_blocks = 0;
  if (Kt != nullptr) {
    const int64_t tiles = pl.n_var * ((pl.kdim_pad + 31) / 32) * ((pl.kc_pad + 31) / 32);
    prep_blocks = std::min<int64_t>(tiles, 2LL * num_sms());
  }
  const int64_t grid = p.n_lower_blocks + prep_blocks;
  if (grid > 0x7FFFFFFF) return cudaErrorInvalidConfiguration;
  if (pl.elt == 2) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(lower_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    lower_kernel<uint16_t><<<static_cast<unsigned>(grid), 256, smem, st>>>(p);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(lower_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    lower_kernel<uint32_t><<<static_cast<unsigned>(grid), 256, smem, st>>>(p);
  }
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace mec
