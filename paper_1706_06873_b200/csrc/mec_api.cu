// mec_api.cu -- the C ABI of libmec.so (include/mec.h): argument validation,
// the host plan (Eq.1, Alg.2 l.8, buffer layout), the stream-ordered
// workspace pool, and the launch sequence of one MEC call:
//   lower(+weight prep) -> window GEMMs -> [Solution A literal format fix].
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <mutex>

#include "../../include/mec.h"
#include "mec_internal.h"
#include "tma_host.h"

namespace mec {
size_t workspace_need(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt, const mec_options_t* opt);
namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

mec_status_t cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorName(e),
           cudaGetErrorString(e));
  return MEC_ERR_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

// One library-owned stream-ordered memory pool per device, with an infinite
// release threshold so repeated calls reuse the same L workspace.
cudaMemPool_t g_pools[kMaxDevices] = {};
std::mutex g_pool_mu;

cudaError_t get_pool(cudaMemPool_t* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    e = cudaMemPoolCreate(&g_pools[dev], &props);
    if (e != cudaSuccess) return e;
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(g_pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = g_pools[dev];
  return cudaSuccess;
}

}  // namespace

int num_sms() {
  static int cached[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  if (cached[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

static cudaError_t encode_impl(CUtensorMap* map, bool tf32, int rank, const void* base,
                               const uint64_t* dims, const uint64_t* strides_bytes,
                               const uint32_t* box, CUtensorMapSwizzle swz,
                               const uint32_t* elem_strides = nullptr);

cudaError_t encode_tiled_strided(CUtensorMap* map, bool tf32, int rank, const void* base,
                                 const uint64_t* dims, const uint64_t* strides_bytes,
                                 const uint32_t* box, const uint32_t* elem_strides) {
  return encode_impl(map, tf32, rank, base, dims, strides_bytes, box, CU_TENSOR_MAP_SWIZZLE_128B,
                     elem_strides);
}

cudaError_t encode_tiled(CUtensorMap* map, bool tf32, int rank, const void* base,
                         const uint64_t* dims, const uint64_t* strides_bytes,
                         const uint32_t* box) {
  return encode_impl(map, tf32, rank, base, dims, strides_bytes, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

cudaError_t encode_tiled_swz(CUtensorMap* map, bool tf32, int rank, const void* base,
                             const uint64_t* dims, const uint64_t* strides_bytes,
                             const uint32_t* box, int swizzle_bytes) {
  const CUtensorMapSwizzle swz = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
  return encode_impl(map, tf32, rank, base, dims, strides_bytes, box, swz);
}

static cudaError_t encode_impl(CUtensorMap* map, bool tf32, int rank, const void* base,
                               const uint64_t* dims, const uint64_t* strides_bytes,
                               const uint32_t* box, CUtensorMapSwizzle swz,
                               const uint32_t* elem_strides) {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  });
  if (!g_encode) return cudaErrorNotSupported;
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5];
  cuuint32_t es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = elem_strides ? elem_strides[i] : 1;
    if (i < rank - 1) s[i] = strides_bytes[i];
  }
  CUresult r = g_encode(map, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                        rank, const_cast<void*>(base), d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Window geometry of the conv-path L for a strip length kw_s >= k_w i_c
// (Alg.2 l.9: row (n, w) of L holds i_h strips; the window of output row h
// starts at column h s_h kw_s), the TMA box alignment, the weight copies and
// the workspace layout.
void set_window_geometry(Plan* p, int64_t kw_s) {
  const mec_shape_t* s = &p->s;
  p->strip = kw_s;
  p->l_cols = s->i_h * kw_s;
  p->kdim = s->k_h * kw_s;
  p->shift = static_cast<int64_t>(p->s_h) * kw_s;
  // box-start alignment: 32 bytes (a 128-byte box row then covers 4 L2
  // sectors, not 5), unless that needs more than 8 shifted weight copies;
  // else the TMA minimum, 16 B
  static const int align_try = getenv("MEC_BOX_ALIGN") ? atoi(getenv("MEC_BOX_ALIGN")) : 32;
  for (int ab : {align_try, 32, 16}) {
    p->avec = ab / p->elt;
    int64_t a = p->shift % p->avec, b = p->avec;  // gcd(shift, avec)
    while (a) { int64_t t = b % a; b = a; a = t; }
    p->delta_step = static_cast<int>(b);
    p->n_var = p->avec / p->delta_step;
    if (p->n_var <= (ab > 32 ? 16 : 8) && p->n_var * p->n_tiles_n <= 32) break;
  }
  p->pitch = round_up(p->l_cols, p->avec);  // row starts keep the box alignment
  p->kdim_pad = round_up(p->kdim + (p->avec - p->delta_step), p->bk);
  if (p->n_var == 1) p->kdim_pad = round_up(p->kdim, p->bk);
  p->bytes_L_pitched = static_cast<size_t>(s->i_n * p->o_w * p->pitch) * p->elt;
  p->off_kt = static_cast<size_t>(round_up(static_cast<int64_t>(p->bytes_L_pitched), 1024));
  p->bytes_kt = static_cast<size_t>(std::max(p->n_var * p->kdim_pad, p->kdim_g) * p->kc_pad) * p->elt;
  // tail: the pair sweep's 3-D weight box reads up to (open rows - 1) window
  // shifts past the last channel row's end (slabs of rows that are not open;
  // never used); open rows <= 7 (at most 8 accumulators, one spare)
  p->bytes_kt += static_cast<size_t>(8 * p->shift + p->bk) * p->elt;
  p->off_wide = static_cast<size_t>(round_up(static_cast<int64_t>(p->off_kt + p->bytes_kt), 1024));
  p->ws_bytes = p->off_kt + p->bytes_kt + 1024;
}

// The atom-major pair sweep where the h-sweep does not apply (its TMEM ring
// cannot hold the window: VGG conv1_2 in tf32) or runs with a single
// accumulator (rows serialised on it: cv8, k_c = 128).  Measured on B200:
// C2 tf32 GEMM 1306 -> 695 us (the one-window kernel before), cv8 b128 337 ->
// 298 us; where the h-sweep has two accumulators it stays faster (C2 bf16 311
// vs 379 us, C3 91 vs 112 us).  MEC_PAIR_SWEEP=1 / 0 forces the choice.
bool pair_sweep_preferred(const Plan& p, bool batch_folded) {
  if (const char* e = getenv("MEC_PAIR_SWEEP")) return atoi(e) != 0;
  int a, n_acc, c, d;
  return !sweep_config(p, batch_folded, &a, &n_acc, &c, &d) || n_acc == 1;
}

Plan strip_padded_plan(const Plan& p) {
  Plan q = p;
  if (p.kwc_s > 0) set_window_geometry(&q, p.kwc_s);
  return q;
}

mec_status_t make_plan(const mec_shape_t* s_in, int s_h, int s_w, mec_dtype_t dt, Plan* p, int pad_h,
                       int pad_w) {
  if (!s_in || !p) return MEC_ERR_INVALID_ARG;
  if (pad_h < 0 || pad_w < 0 || pad_h > (1 << 20) || pad_w > (1 << 20)) return MEC_ERR_INVALID_ARG;
  if (s_in->i_n < 1 || s_in->i_h < 1 || s_in->i_w < 1 || s_in->i_c < 1 || s_in->k_h < 1 ||
      s_in->k_w < 1 || s_in->k_c < 1 || s_h < 1 || s_w < 1)
    return MEC_ERR_INVALID_ARG;
  mec_shape_t padded = *s_in;
  padded.i_h += 2 * static_cast<int64_t>(pad_h);
  padded.i_w += 2 * static_cast<int64_t>(pad_w);
  const mec_shape_t* s = &padded;
  if (s->i_h < s->k_h || s->i_w < s->k_w) return MEC_ERR_INVALID_ARG;
  if (dt != MEC_DTYPE_BF16 && dt != MEC_DTYPE_TF32) return MEC_ERR_INVALID_ARG;
  std::memset(p, 0, sizeof(*p));
  p->s = *s;
  p->pad_h = pad_h;
  p->pad_w = pad_w;
  p->src_h = s_in->i_h;
  p->src_w = s_in->i_w;
  p->s_h = s_h;
  p->s_w = s_w;
  p->dt = dt;
  p->elt = dt == MEC_DTYPE_BF16 ? 2 : 4;
  p->o_h = (s->i_h - s->k_h) / s_h + 1;  // Eq. (1), floor
  p->o_w = (s->i_w - s->k_w) / s_w + 1;
  p->bk = kTileKBytes / p->elt;
  p->vec = 16 / p->elt;
  p->n_tiles_n = static_cast<int>((s->k_c + 255) / 256);
  p->bn = static_cast<int>(round_up((s->k_c + p->n_tiles_n - 1) / p->n_tiles_n, 16));
  p->kc_pad = static_cast<int64_t>(p->n_tiles_n) * p->bn;
  p->n_L = s->i_n * p->o_w * s->i_h * s->k_w * s->i_c;
  p->n_O = s->i_n * p->o_h * p->o_w * s->k_c;
  p->kwc_p = round_up(s->k_w * s->i_c, p->vec);
  p->kdim_g = round_up(s->k_h * p->kwc_p, p->bk);
  p->kdim_src = s->k_h * s->k_w * s->i_c;
  set_window_geometry(p, s->k_w * s->i_c);
  // Strip padding of the conv-path L: when the window shift
  // s_h k_w i_c is not a whole 32-byte MMA K step (AlexNet conv1: 132
  // elements), every strip of k_w i_c elements is stored with kwc_s - k_w i_c
  // zeros after it, kwc_s the smallest length making s_h kwc_s a multiple of
  // 32 bytes.  Then one A stream serves several output rows (multi-row tiles)
  // with one weight copy.  Only where the padding costs <= 15% and windows of
  // neighbouring rows overlap (k_h > s_h).
  {
    const int64_t kwc = s->k_w * s->i_c, step = 32 / p->elt;
    int64_t kw_s = kwc;
    while ((s_h * kw_s) % step != 0 || (kw_s * p->elt) % 2 != 0) ++kw_s;
    if (kw_s != kwc && kw_s * p->elt >= 16 && kw_s * 100 <= kwc * 115 && s->k_h > s_h && p->o_h >= 4 &&
        pad_h == 0 && pad_w == 0 && getenv("MEC_STRIP_PAD")) {
      Plan q = *p;
      set_window_geometry(&q, kw_s);
      p->kwc_s = kw_s;
      p->ws_bytes = std::max(p->ws_bytes, q.ws_bytes);
    }
  }
  // the CTA-pair kernel's scratch (split-K counters and partials) where Alg.2
  // l.8's Solution A would run it automatically (mec_workspace_bytes has no
  // options; resolve() sizes forced cases)
  if (p->kwc_s == 0 && wide_eligible(*p, true, false) && wide_preferred(*p))
    p->ws_bytes = std::max(p->ws_bytes, p->off_wide + wide_scratch_bytes(*p, 0) + 1024);
  // TMA coordinate / extent limits (int32 coordinates, dims <= 2^32)
  if (p->l_cols + p->kdim_pad >= (1LL << 31) || s->i_n * p->o_w >= (1LL << 31) ||
      p->kdim_pad >= (1LL << 31))
    return MEC_ERR_INVALID_ARG;
  return MEC_OK;
}

int select_path_plan(const Plan& p, int T) {
  if (T <= 0) T = MEC_DEFAULT_T;
  // Alg.2 l.8: "if o_w <= T and |O| <= |L|"
  return (p.o_w <= T && p.n_O <= p.n_L) ? MEC_PATH_SOLUTION_A : MEC_PATH_SOLUTION_B;
}

}  // namespace mec

using mec::Plan;

extern "C" {

void mec_options_init(mec_options_t* opt) {
  if (!opt) return;
  std::memset(opt, 0, sizeof(*opt));
  opt->path = MEC_PATH_AUTO;
  opt->T = MEC_DEFAULT_T;
  opt->sola_fix = MEC_SOLA_FIX_EPILOGUE;
}

int mec_abi_version(void) { return MEC_ABI_VERSION; }

const char* mec_status_string(mec_status_t st) {
  switch (st) {
    case MEC_OK: return "MEC_OK";
    case MEC_ERR_INVALID_ARG: return "MEC_ERR_INVALID_ARG";
    case MEC_ERR_UNSUPPORTED: return "MEC_ERR_UNSUPPORTED";
    case MEC_ERR_MISALIGNED: return "MEC_ERR_MISALIGNED";
    case MEC_ERR_CUDA: return "MEC_ERR_CUDA";
    case MEC_ERR_NO_MEMORY: return "MEC_ERR_NO_MEMORY";
  }
  return "MEC_ERR_UNKNOWN";
}

const char* mec_last_error_message(void) { return mec::g_err; }

int mec_last_launch_count(void) { return mec::g_launches; }

mec_status_t mec_out_dims(const mec_shape_t* s, int s_h, int s_w, int64_t* o_h, int64_t* o_w) {
  Plan p;
  if (!o_h || !o_w) return MEC_ERR_INVALID_ARG;
  mec_status_t st = mec::make_plan(s, s_h, s_w, MEC_DTYPE_BF16, &p);
  if (st != MEC_OK) return st;
  *o_h = p.o_h;
  *o_w = p.o_w;
  return MEC_OK;
}

mec_path_t mec_select_path(const mec_shape_t* s, int s_h, int s_w, int T) {
  Plan p;
  if (mec::make_plan(s, s_h, s_w, MEC_DTYPE_BF16, &p) != MEC_OK) return MEC_PATH_AUTO;
  return static_cast<mec_path_t>(mec::select_path_plan(p, T));
}

int64_t mec_lowered_elems(const mec_shape_t* s, int s_h, int s_w) {
  Plan p;
  if (mec::make_plan(s, s_h, s_w, MEC_DTYPE_BF16, &p) != MEC_OK) return -1;
  return p.n_L;
}

int64_t mec_im2col_elems(const mec_shape_t* s, int s_h, int s_w) {
  Plan p;
  if (mec::make_plan(s, s_h, s_w, MEC_DTYPE_BF16, &p) != MEC_OK) return -1;
  return s->i_n * p.o_h * p.o_w * s->k_h * s->k_w * s->i_c;
}

size_t mec_workspace_bytes(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt) {
  Plan p;
  if (mec::make_plan(s, s_h, s_w, dt, &p) != MEC_OK) return 0;
  return p.ws_bytes;
}

size_t mec_workspace_bytes_ex(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt,
                              const mec_options_t* opt) {
  if (!opt) return mec_workspace_bytes(s, s_h, s_w, dt);
  return mec::workspace_need(s, s_h, s_w, dt, opt);
}

mec_status_t mec_lower(const void* I, void* L, const mec_shape_t* s, int s_h, int s_w,
                       mec_dtype_t dt, void* stream) {
  return mec_lower_padded(I, L, s, s_h, s_w, 0, 0, dt, stream);
}

mec_status_t mec_lower_padded(const void* I, void* L, const mec_shape_t* s, int s_h, int s_w,
                              int pad_h, int pad_w, mec_dtype_t dt, void* stream) {
  Plan p;
  mec_status_t st = mec::make_plan(s, s_h, s_w, dt, &p, pad_h, pad_w);
  if (st != MEC_OK) return st;
  if (!I || !L) return MEC_ERR_INVALID_ARG;
  if (!mec::aligned16(I) || !mec::aligned16(L)) return MEC_ERR_MISALIGNED;
  int launches = 0;
  cudaError_t e = mec::launch_lower(p, I, L, p.l_cols, nullptr, nullptr,
                                    static_cast<cudaStream_t>(stream), &launches);
  if (e != cudaSuccess) return mec::cuda_fail(e, "mec_lower");
  mec::g_launches = launches;
  return MEC_OK;
}

mec_status_t mec_lower_pitched(const void* I, void* L, const mec_shape_t* s, int s_h, int s_w,
                               int64_t pitch, mec_dtype_t dt, void* stream) {
  Plan p;
  mec_status_t st = mec::make_plan(s, s_h, s_w, dt, &p, 0, 0);
  if (st != MEC_OK) return st;
  if (!I || !L || pitch < p.l_cols) return MEC_ERR_INVALID_ARG;
  if (!mec::aligned16(I) || !mec::aligned16(L) || (pitch * p.elt) % 16 != 0) return MEC_ERR_MISALIGNED;
  int launches = 0;
  cudaError_t e = mec::launch_lower(p, I, L, pitch, nullptr, nullptr, static_cast<cudaStream_t>(stream),
                                    &launches);
  if (e != cudaSuccess) return mec::cuda_fail(e, "mec_lower_pitched");
  mec::g_launches = launches;
  return MEC_OK;
}

}  // extern "C"

namespace mec {

// Everything one MEC call decides before touching device memory: the plan,
// the path (Alg.2 l.8 or forced), the conv-path plan and the weight-operand
// layout.  Every check that can refuse a call lives here, so callers that
// enqueue several calls (mec_conv_forward_host) can run it up front.
struct Resolved {
  Plan p;          // the (virtually padded) problem
  Plan pc;         // the conv path's plan (strip-padded L where used)
  int path;        // MEC_PATH_SOLUTION_A / _B / _FUSED
  bool gather_kt;  // the fused gather variant's weight-operand layout
  int gemm;        // window-GEMM kernel: 0 = h-sweep if it applies else one window, 1 = one window,
                   // 2 = h-sweep (forced), 3 = CTA pair (split-K), 4 = CTA-pair atom-major sweep
  size_t ws_need;  // workspace bytes this call needs
};

mec_status_t resolve(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt, const mec_options_t* opt,
                     Resolved* r) {
  mec_status_t st = make_plan(s, s_h, s_w, dt, &r->p, opt->pad_h, opt->pad_w);
  if (st != MEC_OK) return st;
  const Plan& p = r->p;
  if (opt->path < MEC_PATH_AUTO || opt->path > MEC_PATH_FASTEST) return MEC_ERR_INVALID_ARG;
  if (opt->sola_fix < MEC_SOLA_FIX_EPILOGUE || opt->sola_fix > MEC_SOLA_FIX_NONE) return MEC_ERR_INVALID_ARG;
  if (opt->rows_per_tile < 0) return MEC_ERR_INVALID_ARG;
  const int T = opt->T > 0 ? opt->T : MEC_DEFAULT_T;
  int path = opt->path;
  if (path == MEC_PATH_FASTEST) {
    // the fused TMA-box variant on the h-sweep, where the layer is not
    // tensor-bound (measured faster there; the one-window and
    // gather variants are not)
    int nv, na, ns, stg;
    const bool paper_wide = wide_preferred(p) && wide_eligible(p, select_path_plan(p, T) != MEC_PATH_SOLUTION_B, false);
    const bool fused_sweep = fused_eligible(p) && !paper_wide && opt->rows_per_tile == 0 &&
                             (opt->gemm_kernel == 0 || opt->gemm_kernel == 2) &&
                             sweep_config(p, true, &nv, &na, &ns, &stg, false);
    path = fused_sweep ? MEC_PATH_FUSED : MEC_PATH_AUTO;
  }
  if (path == MEC_PATH_AUTO) path = select_path_plan(p, T);
  if (path == MEC_PATH_FUSED && !fused_eligible(p) && !gather_eligible(p)) return MEC_ERR_UNSUPPORTED;
  // Solution A's literal format fix repurposes L as auxiliary space,
  // which requires |L| >= |O|.
  if (path == MEC_PATH_SOLUTION_A && opt->sola_fix == MEC_SOLA_FIX_LITERAL && p.n_O > p.n_L)
    return MEC_ERR_UNSUPPORTED;
  r->path = path;
  // the conv path's L: the strip-padded layout where the plan
  // has one and multi-row tiles are not switched off; the fused path reads I
  const bool spad = p.kwc_s > 0 && path != MEC_PATH_FUSED && opt->rows_per_tile != 1;
  r->pc = spad ? strip_padded_plan(p) : p;
  r->gather_kt = path == MEC_PATH_FUSED && !fused_eligible(p);
  if (opt->gemm_kernel < 0 || opt->gemm_kernel > 4 || opt->split_k < 0 || opt->split_k > 64)
    return MEC_ERR_INVALID_ARG;
  const bool batch_folded = path != MEC_PATH_SOLUTION_B;
  const bool wide_ok = !spad && wide_eligible(r->pc, batch_folded, path == MEC_PATH_FUSED) &&
                       opt->sola_fix == MEC_SOLA_FIX_EPILOGUE;
  const bool ps_ok = !spad && pair_sweep_eligible(r->pc, batch_folded, path == MEC_PATH_FUSED);
  if (opt->gemm_kernel == 3) {
    if (!wide_ok) return MEC_ERR_UNSUPPORTED;
    r->gemm = 3;
  } else if (opt->gemm_kernel == 4) {
    if (!ps_ok) return MEC_ERR_UNSUPPORTED;
    r->gemm = 4;
  } else if (opt->gemm_kernel == 0 && opt->rows_per_tile == 0 && wide_ok && wide_preferred(r->pc)) {
    r->gemm = 3;
  } else if (opt->gemm_kernel == 0 && opt->rows_per_tile == 0 && ps_ok && pair_sweep_preferred(r->pc, batch_folded)) {
    r->gemm = 4;
  } else {
    r->gemm = opt->gemm_kernel == 0 ? (opt->rows_per_tile == 0 ? 0 : 1) : opt->gemm_kernel;
  }
  if (r->gemm == 2 && opt->rows_per_tile != 0) return MEC_ERR_INVALID_ARG;
  r->ws_need = p.ws_bytes;
  if (r->gemm == 3)
    r->ws_need = std::max(r->ws_need, r->pc.off_wide + wide_scratch_bytes(r->pc, opt->split_k) + 1024);
  return MEC_OK;
}

size_t workspace_need(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt, const mec_options_t* opt) {
  Resolved r;
  if (resolve(s, s_h, s_w, dt, opt, &r) != MEC_OK) return 0;
  return r.ws_need;
}

// Prepare the weight operand (Alg.2 l.7: K as a (k_h k_w i_c) x k_c matrix,
// K-major, zero padded, shifted copies) into Kt with a prep-only launch.
cudaError_t prepare_weights(const Resolved& r, const void* K, void* Kt, cudaStream_t st, int* launches) {
  if (r.gemm == 3 && wide_reads_k(r.pc)) return cudaSuccess;  // reads K directly
  return launch_lower(r.pc, nullptr, nullptr, r.pc.pitch, K, Kt, st, launches, r.gather_kt);
}

// The launch sequence of one call on a resolved problem: lowering (with the
// weight prep unless kt_ready) -> window GEMMs -> [literal format fix].
cudaError_t run_conv(const Resolved& r, const void* I, const void* K, void* O, void* L, void* Kt, bool kt_ready,
                     cudaStream_t st, mec_options_t* opt, int* launches) {
  const Plan& p = r.p;
  const Plan& pc = r.pc;
  const int path = r.path;
  auto rec = [&](int i) {
    if (opt->stage_events[i]) cudaEventRecord(static_cast<cudaEvent_t>(opt->stage_events[i]), st);
  };
  rec(0);
  // Alg.2 l.2-7: lowering into the pitch-padded L, and K as a (k_h k_w i_c) x k_c matrix
  // (the fused path skips L: only the weight operand is prepared)
  unsigned char* wide_scratch = static_cast<unsigned char*>(L) + pc.off_wide;
  const size_t wide_bytes = r.ws_need - pc.off_wide - 1024;
  // the CTA-pair kernel reads K directly (MN-major B): no weight prep then
  const bool prep = !kt_ready && !(r.gemm == 3 && wide_reads_k(pc));
  cudaError_t e = launch_lower(pc, I, path == MEC_PATH_FUSED ? nullptr : L, pc.pitch, prep ? K : nullptr,
                               prep ? Kt : nullptr, st, launches, r.gather_kt,
                               r.gemm == 3 ? reinterpret_cast<uint32_t*>(wide_scratch) : nullptr,
                               r.gemm == 3 ? wide_zero_words(pc) : 0u);
  if (e != cudaSuccess) return e;
  rec(1);
  GemmArgs ga{};
  ga.L = path == MEC_PATH_FUSED ? I : L;
  ga.fused = path == MEC_PATH_FUSED;
  ga.Kt = Kt;
  ga.K = K;
  ga.O = O;
  ga.rows_per_tile = opt->rows_per_tile;
  if (path == MEC_PATH_FUSED) {  // batch-folded tiles of windows of I
    ga.batch_folded = true;
    ga.out_hnwc = false;
  } else if (path == MEC_PATH_SOLUTION_A) {  // l.9: L as (i_n o_w) x (i_h k_w i_c)
    ga.batch_folded = true;
    ga.out_hnwc = opt->sola_fix != MEC_SOLA_FIX_EPILOGUE;
  } else {  // l.21: L as i_n matrices of o_w x (i_h k_w i_c)
    ga.batch_folded = false;
    ga.out_hnwc = false;
  }
  // r.gemm (resolve): 3 = the CTA-pair kernel; 0 = the h-sweep where it
  // applies, else one window per tile; 1 = one window per tile (R output rows
  // per tile, rows_per_tile); 2 = the h-sweep, forced
  opt->selected_split = 0;
  if (r.gemm == 3) {
    opt->selected_gemm = 3;
    e = launch_wide_gemm(pc, ga, wide_scratch, wide_bytes, opt->split_k, st, launches, &opt->selected_split);
  } else if (r.gemm == 4) {
    opt->selected_gemm = 4;
    e = launch_pair_sweep(pc, ga, st, launches);
  } else {
    e = cudaErrorNotSupported;
    opt->selected_gemm = 2;
    if (r.gemm == 0 || r.gemm == 2) e = launch_sweep_gemm(pc, ga, st, launches);
    if (e == cudaErrorNotSupported && r.gemm != 2) {
      opt->selected_gemm = 1;
      e = launch_window_gemm(pc, ga, st, launches);
    }
  }
  if (e != cudaSuccess) return e;
  rec(2);
  if (path == MEC_PATH_SOLUTION_A && opt->sola_fix == MEC_SOLA_FIX_LITERAL) {
    e = launch_sola_copy(p, O, L, st, launches);  // l.13 Copy L = O
    if (e != cudaSuccess) return e;
    e = launch_sola_transpose(p, L, O, st, launches);  // l.14-19
    if (e != cudaSuccess) return e;
  }
  rec(3);
  opt->selected_path = path;
  return cudaSuccess;
}

}  // namespace mec

extern "C" {

mec_status_t mec_conv_forward_ex(const void* I, const void* K, void* O, const mec_shape_t* s,
                                 int s_h, int s_w, mec_dtype_t dt, void* stream,
                                 mec_options_t* opt) {
  mec_options_t def;
  if (!opt) {
    mec_options_init(&def);
    opt = &def;
  }
  mec::Resolved r;
  mec_status_t st = mec::resolve(s, s_h, s_w, dt, opt, &r);
  if (st != MEC_OK) return st;
  if (!I || !K || !O) return MEC_ERR_INVALID_ARG;
  if (!mec::aligned16(I) || !mec::aligned16(K) || !mec::aligned16(O)) return MEC_ERR_MISALIGNED;
  const Plan& p = r.p;
  cudaStream_t stream_ = static_cast<cudaStream_t>(stream);
  void* ws = opt->workspace;
  bool pooled = false;
  if (ws) {
    if (!mec::aligned16(ws)) return MEC_ERR_MISALIGNED;
    if (opt->workspace_bytes < r.ws_need) return MEC_ERR_NO_MEMORY;
  } else {
    cudaMemPool_t pool;
    cudaError_t e = mec::get_pool(&pool);
    if (e != cudaSuccess) return mec::cuda_fail(e, "mec pool");
    e = cudaMallocFromPoolAsync(&ws, r.ws_need, pool, stream_);
    if (e != cudaSuccess) {
      cudaGetLastError();
      snprintf(mec::g_err, sizeof(mec::g_err), "workspace allocation of %zu bytes failed",
               r.ws_need);
      return MEC_ERR_NO_MEMORY;
    }
    pooled = true;
  }
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(ws) + 1023) & ~static_cast<uintptr_t>(1023));
  int launches = 0;
  const cudaError_t e = mec::run_conv(r, I, K, O, base, base + r.pc.off_kt, false, stream_, opt, &launches);
  if (pooled) cudaFreeAsync(ws, stream_);
  if (e == cudaErrorNotSupported) {  // a forced window-GEMM kernel that cannot run this problem
    snprintf(mec::g_err, sizeof(mec::g_err), "the forced window-GEMM kernel %d does not apply", r.gemm);
    return MEC_ERR_UNSUPPORTED;
  }
  if (e != cudaSuccess) {
    if (getenv("MEC_DEBUG_ERRORS"))
      fprintf(stderr, "mec_conv_forward: failed after %d launches (path %d): %s\n", launches, r.path,
              cudaGetErrorString(e));
    return mec::cuda_fail(e, "mec_conv_forward");
  }
  mec::g_launches = launches;
  return MEC_OK;
}

mec_status_t mec_conv_forward(const void* I, const void* K, void* O, const mec_shape_t* s,
                              int s_h, int s_w, mec_dtype_t dt, void* stream) {
  return mec_conv_forward_ex(I, K, O, s, s_h, s_w, dt, stream, nullptr);
}

mec_status_t mec_maxpool(const void* X, void* Y, int64_t i_n, int64_t h, int64_t w, int64_t c, int p_h,
                         int p_w, int s_h, int s_w, mec_layout_t x_layout, mec_dtype_t dt, void* stream) {
  if (!X || !Y) return MEC_ERR_INVALID_ARG;
  if (i_n < 1 || h < 1 || w < 1 || c < 1 || p_h < 1 || p_w < 1 || s_h < 1 || s_w < 1 || h < p_h ||
      w < p_w)
    return MEC_ERR_INVALID_ARG;
  if (dt != MEC_DTYPE_BF16 && dt != MEC_DTYPE_TF32) return MEC_ERR_INVALID_ARG;
  if (x_layout != MEC_LAYOUT_NHWC && x_layout != MEC_LAYOUT_HNWC) return MEC_ERR_INVALID_ARG;
  const int elt = dt == MEC_DTYPE_BF16 ? 2 : 4;
  if ((c * elt) % 16 != 0) return MEC_ERR_UNSUPPORTED;
  if (!mec::aligned16(X) || !mec::aligned16(Y)) return MEC_ERR_MISALIGNED;
  int launches = 0;
  cudaError_t e = mec::launch_maxpool(X, Y, i_n, h, w, c, p_h, p_w, s_h, s_w, x_layout == MEC_LAYOUT_HNWC,
                                      elt, static_cast<cudaStream_t>(stream), &launches);
  if (e != cudaSuccess) return mec::cuda_fail(e, "mec_maxpool");
  mec::g_launches = launches;
  return MEC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// mec_conv_forward_host: the end-to-end call on host buffers (include/mec.h).
// Chunk c of the images: copy in on the H2D stream, Algorithm 2 on the compute
// stream, copy out on the D2H stream, with a ring of kSlots device buffers so
// the copies of neighbouring chunks overlap chunk c's kernels in both PCIe
// directions.
namespace mec {
namespace {

constexpr int kSlots = 3;

struct HostPipe {
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t start = nullptr, k_in = nullptr;
  cudaEvent_t in[kSlots] = {}, done[kSlots] = {}, out[kSlots] = {};
};
HostPipe g_pipes[kMaxDevices];
std::mutex g_pipe_mu;  // held while a call enqueues (the events are shared)

void destroy_pipe(HostPipe& P) {
  for (cudaStream_t* x : {&P.h2d, &P.comp, &P.d2h})
    if (*x) cudaStreamDestroy(*x);
  for (cudaEvent_t* x : {&P.start, &P.k_in})
    if (*x) cudaEventDestroy(*x);
  for (int i = 0; i < kSlots; ++i)
    for (cudaEvent_t* x : {&P.in[i], &P.done[i], &P.out[i]})
      if (*x) cudaEventDestroy(*x);
  P = HostPipe{};
}

// The device's pipeline (streams + events), created on first use.  It is
// built in a local and published only once every handle exists, so a failed
// creation never leaves a half-built pipeline behind (null streams would be
// the legacy default stream).  Called with g_pipe_mu held.
cudaError_t get_pipe(HostPipe** out) {
  const int dev = current_device();
  HostPipe& P = g_pipes[dev];
  if (!P.h2d) {
    HostPipe q;
    const unsigned ev = cudaEventDisableTiming;
    cudaError_t e = cudaStreamCreateWithFlags(&q.h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&q.comp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&q.d2h, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q.start, ev);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q.k_in, ev);
    for (int i = 0; i < kSlots && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&q.in[i], ev);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q.done[i], ev);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q.out[i], ev);
    }
    if (e != cudaSuccess) {
      destroy_pipe(q);
      return e;
    }
    P = q;
  }
  *out = &P;
  return cudaSuccess;
}

// Byte layout of the device scratch: K | kSlots x (I chunk | O chunk) | workspace.
struct HostLayout {
  int64_t per_chunk, n_chunks, slots;
  size_t i_img, o_img, k_bytes;  // bytes per image of I and O, bytes of K
  size_t off_slot0, slot_bytes, off_o, off_ws, ws_bytes, total;
};

mec_status_t host_layout(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt, const mec_options_t* opt,
                         int n_chunks, HostLayout* h) {
  Plan p;
  mec_status_t st = make_plan(s, s_h, s_w, dt, &p, opt ? opt->pad_h : 0, opt ? opt->pad_w : 0);
  if (st != MEC_OK) return st;
  const int64_t nc = std::min<int64_t>(std::max(n_chunks, 1), s->i_n);
  h->per_chunk = (s->i_n + nc - 1) / nc;
  h->n_chunks = (s->i_n + h->per_chunk - 1) / h->per_chunk;
  h->slots = std::min<int64_t>(kSlots, h->n_chunks);
  h->i_img = static_cast<size_t>(s->i_h * s->i_w * s->i_c) * p.elt;
  h->o_img = static_cast<size_t>(p.o_h * p.o_w * s->k_c) * p.elt;
  h->k_bytes = static_cast<size_t>(s->k_h * s->k_w * s->i_c * s->k_c) * p.elt;
  mec_shape_t sc = *s;
  sc.i_n = h->per_chunk;
  Plan pc;
  st = make_plan(&sc, s_h, s_w, dt, &pc, opt ? opt->pad_h : 0, opt ? opt->pad_w : 0);
  if (st != MEC_OK) return st;
  h->off_slot0 = round_up(h->k_bytes, 1024);
  h->off_o = round_up(h->i_img * h->per_chunk, 1024);
  h->slot_bytes = h->off_o + round_up(h->o_img * h->per_chunk, 1024);
  h->off_ws = h->off_slot0 + h->slots * h->slot_bytes;
  {
    mec_options_t d;
    mec_options_init(&d);
    h->ws_bytes = workspace_need(&sc, s_h, s_w, dt, opt ? opt : &d);
    if (h->ws_bytes == 0) return MEC_ERR_INVALID_ARG;
  }
  h->total = h->off_ws + h->ws_bytes + 1024;  // + alignment slack of the base
  return MEC_OK;
}

}  // namespace
}  // namespace mec

extern "C" {

size_t mec_host_scratch_bytes(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt,
                              const mec_options_t* opt, int n_chunks) {
  mec::HostLayout h;
  if (mec::host_layout(s, s_h, s_w, dt, opt, n_chunks, &h) != MEC_OK) return 0;
  return h.total;
}

mec_status_t mec_conv_forward_host(const void* I_host, const void* K_host, void* O_host,
                                   const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt,
                                   void* stream, mec_options_t* opt, int n_chunks,
                                   void* dev_scratch, size_t dev_scratch_bytes) {
  mec_options_t def;
  if (!opt) {
    mec_options_init(&def);
    opt = &def;
  }
  if (!I_host || !K_host || !O_host) return MEC_ERR_INVALID_ARG;
  mec::HostLayout h;
  mec_status_t st = mec::host_layout(s, s_h, s_w, dt, opt, n_chunks, &h);
  if (st != MEC_OK) return st;
  if (opt->sola_fix == MEC_SOLA_FIX_NONE) return MEC_ERR_UNSUPPORTED;
  // Every check of the per-chunk calls runs here, before anything is enqueued:
  // Alg.2 l.8 on the full shape (forced for every chunk), forced-path
  // eligibility, the literal fix's #O <= #L, rows_per_tile.  (All of them are
  // independent of i_n, so the chunks pass them too.)
  mec::Resolved rf;
  st = mec::resolve(s, s_h, s_w, dt, opt, &rf);
  if (st != MEC_OK) return st;
  mec_options_t co = *opt;
  co.path = rf.path;
  for (auto& ev : co.stage_events) ev = nullptr;
  mec::Resolved rc;  // the full-size chunk (the last one may be smaller)
  {
    mec_shape_t sc = *s;
    sc.i_n = h.per_chunk;
    st = mec::resolve(&sc, s_h, s_w, dt, &co, &rc);
    if (st != MEC_OK) return st;
  }
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  if (dev_scratch) {
    if (!mec::aligned16(dev_scratch)) return MEC_ERR_MISALIGNED;
    if (dev_scratch_bytes < h.total) return MEC_ERR_NO_MEMORY;
  }
  std::lock_guard<std::mutex> lk(mec::g_pipe_mu);
  mec::HostPipe* P = nullptr;
  cudaError_t e = mec::get_pipe(&P);
  if (e != cudaSuccess) return mec::cuda_fail(e, "mec host pipeline");
  bool pooled = false;
  void* scratch = dev_scratch;
  if (!scratch) {
    cudaMemPool_t pool;
    if ((e = mec::get_pool(&pool)) != cudaSuccess) return mec::cuda_fail(e, "mec pool");
    if (cudaMallocFromPoolAsync(&scratch, h.total, pool, user) != cudaSuccess) {
      cudaGetLastError();
      snprintf(mec::g_err, sizeof(mec::g_err), "host-call scratch allocation of %zu bytes failed", h.total);
      return MEC_ERR_NO_MEMORY;
    }
    pooled = true;
  }
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(scratch) + 1023) & ~static_cast<uintptr_t>(1023));
  const unsigned char* Ih = static_cast<const unsigned char*>(I_host);
  unsigned char* Oh = static_cast<unsigned char*>(O_host);
  unsigned char* ws = base + h.off_ws;
  // the weight operand is the same for every chunk: prepared once, after the
  // largest chunk's L in the workspace (a smaller last chunk's L ends earlier)
  void* Kt = ws + rc.pc.off_kt;
  int kernels = 0;
  // the caller's earlier work (and the pool allocation) precede every copy
  e = cudaEventRecord(P->start, user);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(P->h2d, P->start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(P->comp, P->start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(P->d2h, P->start, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(base, K_host, h.k_bytes, cudaMemcpyHostToDevice, P->h2d);
  if (e == cudaSuccess) e = cudaEventRecord(P->k_in, P->h2d);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(P->comp, P->k_in, 0);
  if (e == cudaSuccess) e = mec::prepare_weights(rc, base, Kt, P->comp, &kernels);
  for (int64_t c = 0; c < h.n_chunks && e == cudaSuccess; ++c) {
    const int sl = static_cast<int>(c % h.slots);
    const int64_t n0 = c * h.per_chunk;
    const int64_t nb = std::min<int64_t>(h.per_chunk, s->i_n - n0);
    unsigned char* Id = base + h.off_slot0 + sl * h.slot_bytes;
    unsigned char* Od = Id + h.off_o;
    // copy in: the slot's I is free once chunk c - slots has been computed
    if (c >= h.slots) e = cudaStreamWaitEvent(P->h2d, P->done[sl], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(Id, Ih + n0 * h.i_img, nb * h.i_img, cudaMemcpyHostToDevice, P->h2d);
    if (e == cudaSuccess) e = cudaEventRecord(P->in[sl], P->h2d);
    // compute: needs its I, and the slot's O drained by chunk c - slots' copy out
    if (e == cudaSuccess) e = cudaStreamWaitEvent(P->comp, P->in[sl], 0);
    if (e == cudaSuccess && c >= h.slots) e = cudaStreamWaitEvent(P->comp, P->out[sl], 0);
    if (e != cudaSuccess) break;
    mec::Resolved rk = rc;
    if (nb != h.per_chunk) {
      mec_shape_t sc = *s;
      sc.i_n = nb;
      if ((st = mec::resolve(&sc, s_h, s_w, dt, &co, &rk)) != MEC_OK) break;
    }
    int launches = 0;
    e = mec::run_conv(rk, Id, base, Od, ws, Kt, true, P->comp, &co, &launches);
    kernels += launches;
    if (e == cudaSuccess) e = cudaEventRecord(P->done[sl], P->comp);
    // copy out
    if (e == cudaSuccess) e = cudaStreamWaitEvent(P->d2h, P->done[sl], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(Oh + n0 * h.o_img, Od, nb * h.o_img, cudaMemcpyDeviceToHost, P->d2h);
    if (e == cudaSuccess) e = cudaEventRecord(P->out[sl], P->d2h);
  }
  if (e == cudaSuccess && st == MEC_OK) {
    // the caller's stream waits for the last copy out (the D2H stream is in order)
    e = cudaEventRecord(P->start, P->d2h);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(user, P->start, 0);
  }
  if (e != cudaSuccess || st != MEC_OK) {
    // a failure after the first enqueue: the caller's stream joins all three
    // pipeline streams, so the scratch is not released (nor the call returned
    // to a caller who may free the host buffers) while copies or kernels that
    // were already enqueued can still touch it
    const cudaError_t first = e;
    cudaGetLastError();
    for (cudaStream_t x : {P->h2d, P->comp, P->d2h}) {
      if (cudaEventRecord(P->start, x) == cudaSuccess) cudaStreamWaitEvent(user, P->start, 0);
    }
    cudaStreamSynchronize(user);
    e = first;
  }
  if (pooled) cudaFreeAsync(scratch, user);
  if (st != MEC_OK) return st;
  if (e != cudaSuccess) return mec::cuda_fail(e, "mec_conv_forward_host");
  opt->selected_path = co.selected_path;
  opt->selected_gemm = co.selected_gemm;
  mec::g_launches = kernels;
  return MEC_OK;
}

}  // extern "C"
