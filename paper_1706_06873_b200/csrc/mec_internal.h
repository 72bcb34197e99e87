// mec_internal.h -- host-side plan of one MEC call and the kernel launchers.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/mec.h"

namespace mec {

constexpr int kBM = 128;           // UMMA_M (rows of a window tile; cta_group::1)
constexpr int kTileKBytes = 128;   // one K-tile row = one 128-byte swizzle row
constexpr int kSmemAlign = 1024;   // SWIZZLE_128B atoms need 1024-byte alignment

// Everything derived from (shape, strides, dtype, path) -- Eq.1, the T rule
// of Alg.2 l.8, the window geometry of Alg.2 l.9-12 / l.21-25 and the device
// buffer layout.  Plain host arithmetic.
struct Plan {
  // s is the shape of the (virtually) zero-padded input the convolution runs
  // on: i_h + 2 pad_h, i_w + 2 pad_w (P:41 assumes padding already applied;
  // NEXT-4 applies it inside the lowering instead).  src_h / src_w are the
  // extents of the caller's unpadded I.
  mec_shape_t s;
  int pad_h, pad_w;
  int64_t src_h, src_w;
  int s_h, s_w;
  mec_dtype_t dt;
  int elt;               // bytes per element (2 bf16, 4 tf32/fp32)
  int64_t o_h, o_w;      // Eq. (1)
  // Window geometry of the L the GEMM reads (set_window_geometry).  strip is
  // its strip length: k_w i_c (the paper's dense L), or kwc_s in the
  // strip-padded plan (strip_padded_plan; the extra elements are zeros).
  int64_t strip;
  int64_t kwc_s;         // strip-padded length for the conv path, 0 = not used
  int64_t kdim_src;      // k_h k_w i_c (the paper's reduction length, whatever the strip)
  int64_t l_cols;        // i_h strip: one row of L (Alg.2 l.9 / l.21 "i_h k_w i_c")
  int64_t pitch;         // l_cols rounded up to 16 B (TMA stride rule), elements
  int64_t kdim;          // k_h k_w i_c: GEMM reduction length
  int64_t shift;         // s_h k_w i_c: column offset between output rows
  int bk;                // K-tile in elements (128 B / elt)
  // TMA needs every box to start 16-byte aligned in dim 0, but window h starts
  // at column h*shift.  The box therefore starts at the aligned column
  // x = h*shift - delta, delta = (h*shift) mod avec (avec = 32/elt, or 16/elt
  // when 32 bytes would need more than 8 copies), and the B operand used for
  // that window is K_mat shifted down by delta rows (zero rows above).  delta
  // takes n_var = avec / gcd(shift, avec) values, multiples of delta_step =
  // gcd(shift, avec); Kt holds one copy per value.
  int vec;               // elements per 16 bytes
  int avec;              // box-start alignment of the window GEMM, elements (32 or 16 bytes)
  int delta_step;        // gcd(shift, vec)
  int n_var;             // number of shifted weight copies
  int64_t kdim_pad;      // (kdim + max delta) rounded up to bk
  // gather path: the reduction index is re-laid out as
  // a kwc_p + j (kernel row a, j < k_w i_c), each kernel row padded to 16 bytes
  // (kwc_p elements) so every 16-byte chunk of an A row is one contiguous run of I
  int64_t kwc_p;
  int64_t kdim_g;        // k_h kwc_p rounded up to bk
  int n_tiles_n;         // ceil(k_c / 256)
  int bn;                // N tile (multiple of 16, <= 256)
  int64_t kc_pad;        // n_tiles_n * bn
  int64_t n_L, n_O;      // #L (dense) and #O, elements
  size_t bytes_L_pitched;  // i_n o_w pitch elt
  size_t off_kt;           // workspace offset of the prepared weight operand
  size_t bytes_kt;         // max(n_var kc_pad kdim_pad, kc_pad kdim_g) elt
  size_t off_wide;         // workspace offset of the CTA-pair kernel's scratch (after Kt)
  size_t ws_bytes;         // total workspace (incl. alignment slack)
};

// The plan's window geometry (l_cols, pitch, kdim, shift, box alignment,
// weight copies, workspace) for strip length kw_s.
void set_window_geometry(Plan* p, int64_t kw_s);
// The conv path's plan: p with the strip-padded geometry when p.kwc_s > 0.
Plan strip_padded_plan(const Plan& p);
// Returns MEC_OK and fills *p, or MEC_ERR_INVALID_ARG.
// pad_h / pad_w >= 0: zero padding applied virtually (never materialised).
mec_status_t make_plan(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt, Plan* p, int pad_h = 0,
                       int pad_w = 0);
// Alg.2 l.8 on a plan (the padded shape): 1 = Solution A, 2 = Solution B.
int select_path_plan(const Plan& p, int T);

// ---- kernels (each returns cudaGetLastError() of its launch) ----

// Lowering (Alg.2 l.3-6) into L with row pitch `pitch` elements; optionally,
// in the same launch, the weight operand (Alg.2 l.7, K as a (k_h k_w i_c) x
// k_c matrix), transposed to K-major and shifted:
//   Kt[v][c][j] = K_mat[j - v*delta_step][c]  (0 outside, v < n_var).
// Kt may be null (mec_lower); L may be null (weight prep only, fused path).
// gather_kt: build the gather path's operand instead (one copy, n_var = 1):
//   Kt[c][a kwc_p + j] = K_mat[a k_w i_c + j][c] for j < k_w i_c, 0 otherwise.
// zero_words / n_zero: words the following GEMM needs zeroed (split-K
// counters of the wide kernel), cleared inside the same launch.
cudaError_t launch_lower(const Plan& p, const void* I, void* L, int64_t pitch, const void* K,
                         void* Kt, cudaStream_t st, int* launches, bool gather_kt = false,
                         uint32_t* zero_words = nullptr, uint32_t n_zero = 0);

// Window GEMMs (Alg.2 l.10-12 or l.23-25) on tcgen05.  batch_folded:
// Solution A (rows of several images share one 128-row tile); otherwise
// Solution B (a tile never mixes images).  out_hnwc: store O in h-n-w-c
// (Alg.2 l.10's "O as o_h x i_n o_w k_c") instead of n-h-w-c.
struct GemmArgs {
  const void* L;
  const void* Kt;
  const void* K;      // the caller's K (k_h, k_w, i_c, k_c): K_mat row-major, read directly as an
                      // MN-major B operand by kernels that need no prepared Kt (wide_gemm.cu)
  void* O;
  bool batch_folded;
  bool out_hnwc;
  int rows_per_tile;  // requested multi-row R (0/1 = one output row per tile)
  bool fused;         // A atoms read straight from I (L == I pointer), see DESIGN.md 6.4
};

// The fused path reads each K-atom (a, b, channel block) of a window tile as a
// TMA box of the NHWC input: needs whole 128-byte channel blocks per pixel and
// a pixel traversal stride s_w <= 2 (box rows x s_w <= 256).
bool fused_eligible(const Plan& p);
// Max pooling of a convolution output X (n-h-w-c, or h-n-w-c when hnwc) into
// Y (n-h-w-c), window p_h x p_w, strides s_h, s_w; c elt must be a multiple of 16.
cudaError_t launch_maxpool(const void* X, void* Y, int64_t i_n, int64_t h, int64_t w, int64_t c, int p_h,
                           int p_w, int s_h, int s_w, bool hnwc, int elt, cudaStream_t st, int* launches);

// Fused path for the other layers (e.g. i_c = 3): input rows staged by bulk
// copies, A atoms assembled in smem by builder warps.
bool gather_eligible(const Plan& p);
cudaError_t launch_window_gemm(const Plan& p, const GemmArgs& a, cudaStream_t st, int* launches);

// The same window GEMMs as a sweep along h with A staged in TMEM
// (sweep_gemm.cu): each 128-row tile of L is streamed once per chunk of H
// output rows instead of once per row.  Returns cudaErrorNotSupported (and
// launches nothing) where it does not apply; the caller then runs
// launch_window_gemm.
bool sweep_config(const Plan& p, bool batch_folded, int* n_vres, int* n_acc, int* ns, int* stages,
                  bool pair = false);
cudaError_t launch_sweep_gemm(const Plan& p, const GemmArgs& a, cudaStream_t st, int* launches);

// Window GEMMs of the tensor-bound layers on CTA pairs (wide_gemm.cu):
// tcgen05 cta_group::2 (M = 256), split-K across pairs with an in-order
// reduction.  Solution A with flat rows (o_w < 32) only.
bool wide_eligible(const Plan& p, bool batch_folded, bool fused);
bool wide_preferred(const Plan& p);  // tensor-bound (AI >= 0.8 ridge) or MEC_WIDE
// the CTA-pair kernel reads the weights straight from K (MN-major B, no Kt)
bool wide_reads_k(const Plan& p);
// scratch (counters + fp32 partials) for split `split` (0 = automatic)
size_t wide_scratch_bytes(const Plan& p, int split);
// words of the scratch that must be zero when the kernel starts
uint32_t wide_zero_words(const Plan& p);
cudaError_t launch_wide_gemm(const Plan& p, const GemmArgs& a, void* scratch, size_t scratch_bytes, int split,
                             cudaStream_t st, int* launches, int* split_used);

// Window GEMMs as an atom-major sweep along h on CTA pairs (pair_sweep.cu):
// windows starting on 128-byte atom boundaries (shift a whole number of
// atoms), any window width, weights resident (k_c / 2 rows per CTA).
bool pair_sweep_eligible(const Plan& p, bool batch_folded, bool fused);
cudaError_t launch_pair_sweep(const Plan& p, const GemmArgs& a, cudaStream_t st, int* launches);

// Solution A format fix, paper-literal (Alg.2 l.13-19): "Copy L = O" and the
// block transpose O[n,h,:] = L[h,n,:].
cudaError_t launch_sola_copy(const Plan& p, const void* O, void* Laux, cudaStream_t st,
                             int* launches);
cudaError_t launch_sola_transpose(const Plan& p, const void* Laux, void* O, cudaStream_t st,
                                  int* launches);

int num_sms();

// Per-device library state (pools, host pipelines, kernel attributes) is kept
// in arrays of kMaxDevices; current_device() clamps the ordinal into them.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

}  // namespace mec
