// pool.cu -- max pooling that consumes a convolution output in n-h-w-c or in
// Solution A's h-n-w-c ("if the following layer is
// pooling, ... the output in h-n-w-c can be consumed directly", so Solution
// A's transpose, Alg.2 l.13-19, is skipped).
//
// Y[n, y, x, c] = max over (dy, dx) < (p_h, p_w) of X[n, y s_h + dy, x s_w + dx, c]
// with X read in either layout and Y written in n-h-w-c.  Memory-bound: one
// thread per 16-byte channel vector of one output pixel (8 bf16 / 4 fp32),
// consecutive threads on consecutive vectors, so every load and store is a
// coalesced 128-bit access; bf16 maxima are exact (__hmax2).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mec_internal.h"

namespace mec {
namespace {

struct PoolParams {
  const unsigned char* X;
  unsigned char* Y;
  int64_t i_n, h, w, c;      // X extents
  int64_t o_h, o_w;          // Y extents (floor, Eq. 1 form)
  int p_h, p_w, s_h, s_w;
  bool hnwc;                 // X in h-n-w-c
  int64_t vecs_per_pixel;    // c / elements per 16 bytes
};

__device__ __forceinline__ uint4 vmax(uint4 a, uint4 b, bool bf16) {
  if (bf16) {
    auto m = [](uint32_t x, uint32_t y) {
      __nv_bfloat162 r = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&x), *reinterpret_cast<__nv_bfloat162*>(&y));
      return *reinterpret_cast<uint32_t*>(&r);
    };
    return make_uint4(m(a.x, b.x), m(a.y, b.y), m(a.z, b.z), m(a.w, b.w));
  }
  return make_uint4(__float_as_uint(fmaxf(__uint_as_float(a.x), __uint_as_float(b.x))),
                    __float_as_uint(fmaxf(__uint_as_float(a.y), __uint_as_float(b.y))),
                    __float_as_uint(fmaxf(__uint_as_float(a.z), __uint_as_float(b.z))),
                    __float_as_uint(fmaxf(__uint_as_float(a.w), __uint_as_float(b.w))));
}

template <bool kBF16>
__global__ void __launch_bounds__(256) maxpool_kernel(const PoolParams p) {
  const int64_t total = p.i_n * p.o_h * p.o_w * p.vecs_per_pixel;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = i % p.vecs_per_pixel;
    int64_t r = i / p.vecs_per_pixel;
    const int64_t x = r % p.o_w;
    r /= p.o_w;
    const int64_t y = r % p.o_h;
    const int64_t n = r / p.o_h;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int dy = 0; dy < p.p_h; ++dy) {
      const int64_t yy = y * p.s_h + dy;
      for (int dx = 0; dx < p.p_w; ++dx) {
        const int64_t xx = x * p.s_w + dx;
        // pixel (n, yy, xx) of X: n-h-w-c or h-n-w-c
        const int64_t pix = p.hnwc ? (yy * p.i_n + n) * p.w + xx : (n * p.h + yy) * p.w + xx;
        const uint4 val = __ldg(reinterpret_cast<const uint4*>(p.X) + pix * p.vecs_per_pixel + v);
        acc = (dy == 0 && dx == 0) ? val : vmax(acc, val, kBF16);
      }
    }
    reinterpret_cast<uint4*>(p.Y)[i] = acc;
  }
}

}  // namespace

cudaError_t launch_maxpool(const void* X, void* Y, int64_t i_n, int64_t h, int64_t w, int64_t c, int p_h,
                           int p_w, int s_h, int s_w, bool hnwc, int elt, cudaStream_t st, int* launches) {
  PoolParams p{};
  p.X = static_cast<const unsigned char*>(X);
  p.Y = static_cast<unsigned char*>(Y);
  p.i_n = i_n;
  p.h = h;
  p.w = w;
  p.c = c;
  p.p_h = p_h;
  p.p_w = p_w;
  p.s_h = s_h;
  p.s_w = s_w;
  p.o_h = (h - p_h) / s_h + 1;
  p.o_w = (w - p_w) / s_w + 1;
  p.hnwc = hnwc;
  p.vecs_per_pixel = c * elt / 16;
  const int64_t total = i_n * p.o_h * p.o_w * p.vecs_per_pixel;
  if (total == 0) return cudaSuccess;
  const int64_t grid = std::min<int64_t>((total + 255) / 256, 64LL * num_sms());
  if (elt == 2)
    maxpool_kernel<true><<<static_cast<unsigned>(grid), 256, 0, st>>>(p);
  else
    maxpool_kernel<false><<<static_cast<unsigned>(grid), 256, 0, st>>>(p);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace mec
