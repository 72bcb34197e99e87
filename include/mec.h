/*
 * mec.h -- C ABI of libmec.so, the B200 (sm_100a) hot path of MEC
 * (Cho & Brand, "MEC: Memory-efficient Convolution for Deep Neural Network",
 *  ICML 2017, arXiv 1706.06873).  "P:<n>" cites line n of the paper text.
 *
 * The operation (Sec. 2.1): O = I * K with strides s_h, s_w; zero
 * padding is assumed already applied to I; o = (i - k) / s + 1 (Eq. 1, floor).
 * Layouts (Table 1), all row-major:
 *   I  i_n x i_h x i_w x i_c     (n-h-w-c)
 *   K  k_h x k_w x i_c x k_c     (read as a (k_h k_w i_c) x k_c matrix, Alg.2 l.7)
 *   O  i_n x o_h x o_w x k_c     (n-h-w-c, Alg.2 l.27)
 *   L  i_n x o_w x i_h x k_w x i_c  (MEC's compact lowered tensor, Alg.2 l.2-6)
 *
 * Conventions for every entry point:
 *  - All tensor pointers are DEVICE pointers owned by the caller (except the
 *    HOST buffers of mec_conv_forward_host).  The library
 *    never frees or retains them past the call; work is enqueued
 *    asynchronously on `stream` (a cudaStream_t; NULL = legacy default
 *    stream), so buffers must stay alive until the stream reaches the work.
 *  - Functions never throw and never abort; they return an mec_status_t.
 *    On MEC_ERR_CUDA the CUDA error string is available from
 *    mec_last_error_message() (per-thread).
 *  - I, O and L must not alias each other.  I and K are read-only.
 *  - dtype: MEC_DTYPE_BF16 -> I, K, O are bf16 (2 B), fp32 accumulation in
 *    tensor memory, O rounded to nearest-even.  MEC_DTYPE_TF32 -> I, K, O are
 *    fp32 (4 B) in memory, multiplied as tf32 (tcgen05 kind::tf32), fp32
 *    accumulation, O written as fp32.
 *  - Inputs must be finite: the K-tail of a window reads up to one K-tile of
 *    neighbouring lowered data, multiplied by zero weight rows.
 */
#ifndef MEC_H
#define MEC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MEC_ABI_VERSION 6

typedef enum {
  MEC_OK = 0,
  MEC_ERR_INVALID_ARG = 1, /* extent < 1, stride < 1, i < k, NULL pointer, bad enum */
  MEC_ERR_UNSUPPORTED = 2, /* forced path infeasible (e.g. Solution A with #O > #L) */
  MEC_ERR_MISALIGNED = 3,  /* I, K, O, L or workspace not 16-byte aligned */
  MEC_ERR_CUDA = 4,        /* a CUDA runtime / driver error; see mec_last_error_message() */
  MEC_ERR_NO_MEMORY = 5    /* workspace too small, or the stream-ordered allocation failed */
} mec_status_t;

typedef enum {
  MEC_DTYPE_BF16 = 0,
  MEC_DTYPE_TF32 = 1
} mec_dtype_t;

/* Table 1 symbols.  k_c is the number of output channels. */
typedef struct {
  int64_t i_n, i_h, i_w, i_c, k_h, k_w, k_c;
} mec_shape_t;

/* Which of Algorithm 2's two solutions runs.  The paper's letters
 * are used: Solution A = batch-folded GEMMs (o_h GEMMs of (i_n o_w) rows,
 * Alg.2 l.9-19); Solution B = per-image GEMMs (i_n o_h GEMMs of o_w rows,
 * Alg.2 l.20-25).  (BASELINE.json's north_star swaps the two letters.) */
typedef enum {
  MEC_PATH_AUTO = 0,       /* Alg.2 l.8: A iff o_w <= T and #O <= #L, else B */
  MEC_PATH_SOLUTION_A = 1, /* batch-folded */
  MEC_PATH_SOLUTION_B = 2, /* per-image */
  MEC_PATH_FUSED = 3,      /* lowering fused into the GEMM: each K-atom of a window tile is
                              read as a TMA box of I, L is never written (needs i_c elt a
                              multiple of 128 B and s_w <= 2; else MEC_ERR_UNSUPPORTED).
                              Never chosen by MEC_PATH_AUTO (which follows Alg.2 l.8). */
  MEC_PATH_FASTEST = 4     /* MEC_PATH_FUSED where its TMA-box variant runs as the h-sweep
                              and the layer is not tensor-bound (measured faster on B200:
                              VGG conv1_2 b64 301 vs 563 us, ResNet-50 3x3 b256 101 vs 159,
                              cv8 / cv9 1.25-1.6x), else MEC_PATH_AUTO's choice.  Not a
                              paper rule: the paper's path (Alg.2 l.8) is MEC_PATH_AUTO. */
} mec_path_t;

/* How Solution A reaches n-h-w-c (Alg.2 l.13-19). */
typedef enum {
  MEC_SOLA_FIX_EPILOGUE = 0, /* GEMM epilogue stores O[n,h] = O_hnwc[h,n] directly (default) */
  MEC_SOLA_FIX_LITERAL = 1,  /* paper-literal: GEMMs write O in h-n-w-c, "Copy L = O",
                                then O[n,h,:] = L[h,n,:] (two extra passes over O) */
  MEC_SOLA_FIX_NONE = 2      /* leave O in h-n-w-c (a following pooling layer may
                                consume h-n-w-c); O is then o_h x i_n x o_w x k_c */
} mec_sola_fix_t;

#define MEC_DEFAULT_T 100 /* "we found T around 100 to be a good threshold" */

typedef struct {
  int path;       /* mec_path_t; MEC_PATH_AUTO by default */
  int T;          /* threshold of Alg.2 l.8; <= 0 means MEC_DEFAULT_T */
  int sola_fix;   /* mec_sola_fix_t; used only when Solution A runs */
  int rows_per_tile; /* 0 = auto: the h-sweep window GEMM where it applies (each
                        128-row tile of L streamed once per chunk of output rows,
                        DESIGN.md 6.2b), else the one-window-per-tile kernel with its
                        automatic rows per tile.  >= 1: force the one-window-per-tile
                        kernel with this many output rows h per tile (the union of
                        their overlapping windows of L is streamed once). */
  void* workspace;        /* device buffer >= mec_workspace_bytes(); NULL = stream-ordered pool */
  size_t workspace_bytes;
  /* Optional cudaEvent_t handles recorded on `stream` at stage boundaries
   * (NULL entries are skipped): [0] before lowering, [1] after lowering,
   * [2] after the window GEMMs, [3] after the Solution A format fix (== [2]
   * when there is none).  For per-stage timing only. */
  void* stage_events[4];
  int selected_path; /* OUT: the path that ran (1 = A, 2 = B, 3 = fused) */
  /* Zero padding: the convolution runs on I padded with
   * pad_h zero rows above and below and pad_w zero columns left and right
   * (P:41 assumes this padding already applied to I).  The padded input is
   * never materialised: the lowering (or the fused path's TMA zero fill)
   * produces the lowered rows of the padded image directly.  o from Eq. 1 on
   * the padded extents; O is i_n x o_h x o_w x k_c of the padded problem.
   * Not supported by the fused gather variant (MEC_ERR_UNSUPPORTED). */
  int pad_h, pad_w;
  int selected_gemm; /* OUT: the window-GEMM kernel that ran: 1 = one window per tile
                        (DESIGN.md 6.2), 2 = h-sweep with A in TMEM (6.2b), 3 = CTA-pair
                        (cta_group::2) kernel with split-K (6.7), 4 = CTA-pair atom-major
                        sweep (6.8), 0 = none */
  /* ABI version 5.  gemm_kernel (IN) forces the window-GEMM kernel: 0 = automatic
   * (the CTA-pair kernel for tensor-bound Solution A layers with o_w < 32, else
   * the h-sweep where it applies, else the CTA-pair atom-major sweep where it
   * applies, else one window per tile), 1 = one window per tile, 2 = h-sweep,
   * 3 = CTA pair with split-K, 4 = CTA-pair atom-major sweep.  A forced kernel that cannot run the
   * problem returns MEC_ERR_UNSUPPORTED.  split_k (IN): K ranges of the CTA-pair
   * kernel, 0 = automatic (1..8 by a wave model); the ranges' fp32 partials are
   * summed in range order, so the result depends on split_k but not on timing.
   * selected_split (OUT): the split the CTA-pair kernel used (0 otherwise). */
  int gemm_kernel;
  int split_k;
  int selected_split;
} mec_options_t;

/* Fills *opt with defaults (AUTO path, T = 100, epilogue fix, pool workspace). */
void mec_options_init(mec_options_t* opt);

/* Eq. (1), P:43 with floor (reading Q1).  MEC_ERR_INVALID_ARG on a
 * bad shape or NULL output pointer. */
mec_status_t mec_out_dims(const mec_shape_t* s, int s_h, int s_w, int64_t* o_h,
                          int64_t* o_w);

/* Alg.2 l.8: MEC_PATH_SOLUTION_A iff o_w <= T and
 * #O <= #L, else MEC_PATH_SOLUTION_B.  T <= 0 means 100.  Host-only; returns
 * MEC_PATH_AUTO (0) for an invalid shape. */
mec_path_t mec_select_path(const mec_shape_t* s, int s_h, int s_w, int T);

/* Closed-form element counts: #L_MEC = i_n o_w i_h k_w i_c (Table 1, Alg.2
 * l.2), #L_im2col = i_n o_h o_w k_h k_w i_c (Eq. 2 with i_c, reading Q2).
 * Return -1 for an invalid shape. */
int64_t mec_lowered_elems(const mec_shape_t* s, int s_h, int s_w);
int64_t mec_im2col_elems(const mec_shape_t* s, int s_h, int s_w);

/* Bytes of device workspace mec_conv_forward_ex needs for this problem:
 * the pitch-padded lowered tensor L (i_n o_w rows of i_h k_w i_c elements,
 * row pitch rounded up to 16 B), the prepared weight operand and alignment
 * slack.  Never an im2col-sized buffer.  0 for an invalid shape/dtype. */
size_t mec_workspace_bytes(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt);

/* Compact lowering, Alg.2 l.3-6:
 *   L[n, w, h, 0:k_w, 0:i_c] = I[n, h, s_w w : s_w w + k_w, 0:i_c]
 * for all n < i_n, w < o_w, h < i_h (every input row, reading Q5).  L is the
 * DENSE paper layout (#L = i_n o_w i_h k_w i_c elements), a bit-exact copy of
 * I's elements.  Only the element size of dt matters (2 B bf16, 4 B tf32).
 * I and L need 16-byte alignment. */
mec_status_t mec_lower(const void* I, void* L, const mec_shape_t* s, int s_h,
                       int s_w, mec_dtype_t dt, void* stream);

/* mec_workspace_bytes for the padded problem of opt->pad_h / opt->pad_w
 * (opt may be NULL = no padding). */
size_t mec_workspace_bytes_ex(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt,
                              const mec_options_t* opt);

/* Compact lowering of the zero-padded input (NEXT-4): s holds the UNPADDED
 * extents of I; L is the dense lowering of the (i_h + 2 pad_h) x
 * (i_w + 2 pad_w) padded image, i_n x o_w x (i_h + 2 pad_h) x k_w x i_c,
 * with zeros wherever the padded image is zero.  pad_h = pad_w = 0 is
 * mec_lower.  Errors as mec_lower (negative pads: MEC_ERR_INVALID_ARG). */
mec_status_t mec_lower_padded(const void* I, void* L, const mec_shape_t* s, int s_h, int s_w,
                              int pad_h, int pad_w, mec_dtype_t dt, void* stream);

/* Compact lowering into a caller-chosen row pitch (ABI 3): as mec_lower, but
 * row (n, w) of L (its i_h k_w i_c elements, Alg.2 l.9's L matrix row) starts
 * at element (n o_w + w) * pitch; the pitch - i_h k_w i_c trailing elements
 * of a row are unspecified on return (they may be overwritten).  This is the
 * layout the conv path lowers into (pitch = i_h k_w i_c rounded up to 16
 * bytes, the TMA stride rule), exposed so it can be checked bit for bit.
 * pitch < i_h k_w i_c: MEC_ERR_INVALID_ARG; pitch elt not a multiple of 16 B:
 * MEC_ERR_MISALIGNED. */
mec_status_t mec_lower_pitched(const void* I, void* L, const mec_shape_t* s, int s_h, int s_w,
                               int64_t pitch, mec_dtype_t dt, void* stream);

/* O = MEC(I, K, s) (Algorithm 2): lowering, then the window GEMMs
 * of the path picked by Alg.2 l.8 with T = 100, then (Solution A) the format
 * fix, all on `stream`.  O receives i_n x o_h x o_w x k_c in n-h-w-c.  L is
 * taken from a stream-ordered pool (Alg.2 l.2 allocates L inside MEC). */
mec_status_t mec_conv_forward(const void* I, const void* K, void* O,
                              const mec_shape_t* s, int s_h, int s_w,
                              mec_dtype_t dt, void* stream);

/* As mec_conv_forward, with a forced path / threshold / Solution-A format fix
 * / caller workspace / stage events (opt may be NULL = defaults). */
mec_status_t mec_conv_forward_ex(const void* I, const void* K, void* O,
                                 const mec_shape_t* s, int s_h, int s_w,
                                 mec_dtype_t dt, void* stream,
                                 mec_options_t* opt);

/* End to end on HOST buffers (ABI 4): O_host = MEC(I_host, K_host, s), the
 * same Algorithm 2 call as mec_conv_forward_ex with the
 * host<->device copies inside.  The i_n images are cut into n_chunks chunks of
 * ceil(i_n / n_chunks) images (each chunk is an independent convolution of a
 * sub-batch: Alg.2 never mixes images); chunk c's copy in, its MEC call and
 * its copy out run on three library streams so the copy in of chunk c + 1 and
 * the copy out of chunk c - 1 overlap chunk c's kernels (the PCIe link is
 * full duplex).  The path is resolved ONCE on the full shape (Alg.2 l.8 with
 * opt->T) and forced for every chunk, so each image takes the path the
 * one-shot call would take.
 *   I_host  i_n x i_h x i_w x i_c, K_host k_h x k_w x i_c x k_c, O_host
 *           i_n x o_h x o_w x k_c, all n-h-w-c, caller-owned host memory.
 *           Page-locked (cudaHostAlloc / torch pin_memory) for the copies to
 *           be asynchronous; pageable memory works but serialises them.
 *   stream  the caller's stream: work already on it is ordered before the
 *           first copy, and it waits for the last copy out, so O_host is
 *           complete once `stream` is synchronised.
 *   opt     as mec_conv_forward_ex (NULL = defaults); opt->workspace is
 *           ignored (the scratch holds it); MEC_SOLA_FIX_NONE is
 *           MEC_ERR_UNSUPPORTED (h-n-w-c is not contiguous per chunk).
 *   dev_scratch  device buffer of >= mec_host_scratch_bytes(...) bytes,
 *           16-byte aligned, caller-owned, not touched after `stream`
 *           completes; NULL = taken from the library's stream-ordered pool.
 * n_chunks < 1 or > i_n: clamped to [1, i_n].  Errors as mec_conv_forward_ex;
 * a copy failure is MEC_ERR_CUDA.  mec_last_launch_count() afterwards is the
 * number of KERNELS enqueued over all chunks (copies are not counted). */
size_t mec_host_scratch_bytes(const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt,
                              const mec_options_t* opt, int n_chunks);
mec_status_t mec_conv_forward_host(const void* I_host, const void* K_host, void* O_host,
                                   const mec_shape_t* s, int s_h, int s_w, mec_dtype_t dt,
                                   void* stream, mec_options_t* opt, int n_chunks,
                                   void* dev_scratch, size_t dev_scratch_bytes);

/* Layout of a convolution output consumed by mec_maxpool. */
typedef enum {
  MEC_LAYOUT_NHWC = 0, /* i_n x h x w x c (Alg.2 l.27's O) */
  MEC_LAYOUT_HNWC = 1  /* h x i_n x w x c (Solution A's O before l.13-19, MEC_SOLA_FIX_NONE) */
} mec_layout_t;

/* Max pooling as the consumer of a convolution output (
 * a following pooling layer can consume Solution A's h-n-w-c output,
 * so its transpose is skipped):
 *   Y[n, y, x, :] = max_{dy < p_h, dx < p_w} X[n, y s_h + dy, x s_w + dx, :]
 * X has extents (i_n, h, w, c) in x_layout; Y is n-h-w-c, i_n x
 * ((h - p_h)/s_h + 1) x ((w - p_w)/s_w + 1) x c (floor).  Device pointers,
 * 16-byte aligned; c elt must be a multiple of 16 bytes (else
 * MEC_ERR_UNSUPPORTED).  bf16 maxima are exact; fp32 uses fmaxf. */
mec_status_t mec_maxpool(const void* X, void* Y, int64_t i_n, int64_t h, int64_t w, int64_t c,
                         int p_h, int p_w, int s_h, int s_w, mec_layout_t x_layout, mec_dtype_t dt,
                         void* stream);

/* Number of kernel launches the last successful conv / lower call on this
 * thread enqueued (for the bench's gpu_launches count). */
int mec_last_launch_count(void);

const char* mec_status_string(mec_status_t st);
const char* mec_last_error_message(void);
int mec_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MEC_H */
