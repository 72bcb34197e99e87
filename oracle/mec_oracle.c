/*
 * mec_oracle.c -- plain C11 CPU oracle for MEC (arXiv 1706.06873).
 *
 * TEST INFRASTRUCTURE ONLY (see mec_oracle.h).  Written from PAPER.md; each
 * function cites the passage it follows.  No blocking, fusion, SIMD or BLAS:
 * every loop is the definition or the algorithm step, in the paper's order.
 * Accumulation is in double.  Threads (pthreads) only split independent
 * images n, which Alg.2 runs "in parallel" (l.4, l.17, l.22).
 */
#include "mec_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- shapes */

static int shape_ok(const mec_oracle_shape* s, int s_h, int s_w) {
  if (!s) return 0;
  if (s->i_n < 1 || s->i_h < 1 || s->i_w < 1 || s->i_c < 1) return 0;
  if (s->k_h < 1 || s->k_w < 1 || s->k_c < 1) return 0;
  if (s_h < 1 || s_w < 1) return 0;
  if (s->i_h < s->k_h || s->i_w < s->k_w) return 0;
  return 1;
}

/* Eq. (1).  Zero padding is already applied to I, so there
 * is no padding argument.  When s does not divide i - k the floor is taken
 * (reading Q1, pinned by Table 3 cv4 in tests/golden/table3_resnet101.txt). */
int mec_oracle_out_dims(const mec_oracle_shape* s, int s_h, int s_w,
                        int64_t* o_h, int64_t* o_w) {
  if (!shape_ok(s, s_h, s_w)) return -1;
  if (o_h) *o_h = (s->i_h - s->k_h) / s_h + 1;
  if (o_w) *o_w = (s->i_w - s->k_w) / s_w + 1;
  return 0;
}

/* Table 1 L is i_n x o_w x i_h x k_w x i_c; Alg.2 l.2. */
int64_t mec_oracle_elems_L_mec(const mec_oracle_shape* s, int s_h, int s_w) {
  int64_t oh, ow;
  if (mec_oracle_out_dims(s, s_h, s_w, &oh, &ow)) return -1;
  return s->i_n * ow * s->i_h * s->k_w * s->i_c;
}

/* Eq. (2): i_n o_h o_w x k_h k_w (i_c) -- one row per window. */
int64_t mec_oracle_elems_L_im2col(const mec_oracle_shape* s, int s_h, int s_w) {
  int64_t oh, ow;
  if (mec_oracle_out_dims(s, s_h, s_w, &oh, &ow)) return -1;
  return s->i_n * oh * ow * s->k_h * s->k_w * s->i_c;
}

/* Alg.2 l.1: O has i_n o_h o_w k_c elements. */
int64_t mec_oracle_elems_O(const mec_oracle_shape* s, int s_h, int s_w) {
  int64_t oh, ow;
  if (mec_oracle_out_dims(s, s_h, s_w, &oh, &ow)) return -1;
  return s->i_n * oh * ow * s->k_c;
}

/* Alg.2 l.8: "if o_w <= T and |O| <= |L| then" Solution A else B. */
int mec_oracle_select_path(const mec_oracle_shape* s, int s_h, int s_w, int T) {
  int64_t oh, ow;
  if (mec_oracle_out_dims(s, s_h, s_w, &oh, &ow)) return -1;
  int64_t nO = mec_oracle_elems_O(s, s_h, s_w);
  int64_t nL = mec_oracle_elems_L_mec(s, s_h, s_w);
  return (ow <= (int64_t)T && nO <= nL) ? 1 : 2;
}

/* ------------------------------------------------------- image threading */

typedef struct {
  void (*fn)(void* ctx, int64_t n);
  void* ctx;
  int64_t n_begin, n_end;
} img_range;

static void* img_worker(void* arg) {
  img_range* r = (img_range*)arg;
  for (int64_t n = r->n_begin; n < r->n_end; ++n) r->fn(r->ctx, n);
  return NULL;
}

/* Runs fn(ctx, n) for every image n in [0, i_n), images split over threads. */
static void for_each_image(int64_t i_n, int n_threads,
                           void (*fn)(void*, int64_t), void* ctx) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > i_n) n_threads = (int)i_n;
  if (n_threads <= 1) {
    for (int64_t n = 0; n < i_n; ++n) fn(ctx, n);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  img_range* rg = (img_range*)malloc(sizeof(img_range) * (size_t)n_threads);
  for (int t = 0; t < n_threads; ++t) {
    rg[t].fn = fn;
    rg[t].ctx = ctx;
    rg[t].n_begin = i_n * t / n_threads;
    rg[t].n_end = i_n * (t + 1) / n_threads;
    pthread_create(&th[t], NULL, img_worker, &rg[t]);
  }
  for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(rg);
}

/* -------------------------------------------------------- direct conv */

typedef struct {
  const double *I, *K;
  double* O;
  const mec_oracle_shape* s;
  int s_h, s_w;
  int64_t o_h, o_w;
} conv_ctx;

/* Fig. 1(a): each O element is the dot product of K with the
 * sub-matrix of I at (h s_h, w s_w); no kernel flip (reading Q3). */
static void direct_conv_image(void* vctx, int64_t n) {
  const conv_ctx* c = (const conv_ctx*)vctx;
  const mec_oracle_shape* s = c->s;
  for (int64_t h = 0; h < c->o_h; ++h)
    for (int64_t w = 0; w < c->o_w; ++w)
      for (int64_t kc = 0; kc < s->k_c; ++kc) {
        double acc = 0.0;
        for (int64_t a = 0; a < s->k_h; ++a)
          for (int64_t b = 0; b < s->k_w; ++b)
            for (int64_t ci = 0; ci < s->i_c; ++ci) {
              int64_t y = h * c->s_h + a, x = w * c->s_w + b;
              double iv = c->I[((n * s->i_h + y) * s->i_w + x) * s->i_c + ci];
              double kv = c->K[((a * s->k_w + b) * s->i_c + ci) * s->k_c + kc];
              acc += iv * kv;
            }
        c->O[((n * c->o_h + h) * c->o_w + w) * s->k_c + kc] = acc;
      }
}

int mec_oracle_direct_conv(const double* I, const double* K, double* O,
                           const mec_oracle_shape* s, int s_h, int s_w,
                           int n_threads) {
  conv_ctx c = {I, K, O, s, s_h, s_w, 0, 0};
  if (!I || !K || !O) return -1;
  if (mec_oracle_out_dims(s, s_h, s_w, &c.o_h, &c.o_w)) return -1;
  for_each_image(s->i_n, n_threads, direct_conv_image, &c);
  return 0;
}

/* ------------------------------------------------------------- im2col */

/* Fig. 1(b): "each sub-matrix instance w.r.t. K is linearized into a
 * row of the lowered matrix"; Eq. (2) gives its dimensions. */
int mec_oracle_im2col(const double* I, double* C, const mec_oracle_shape* s,
                      int s_h, int s_w) {
  int64_t oh, ow;
  if (!I || !C || mec_oracle_out_dims(s, s_h, s_w, &oh, &ow)) return -1;
  const int64_t cols = s->k_h * s->k_w * s->i_c;
  for (int64_t n = 0; n < s->i_n; ++n)
    for (int64_t h = 0; h < oh; ++h)
      for (int64_t w = 0; w < ow; ++w) {
        int64_t row = (n * oh + h) * ow + w;
        for (int64_t a = 0; a < s->k_h; ++a)
          for (int64_t b = 0; b < s->k_w; ++b)
            for (int64_t ci = 0; ci < s->i_c; ++ci) {
              int64_t col = (a * s->k_w + b) * s->i_c + ci;
              C[row * cols + col] =
                  I[((n * s->i_h + h * s_h + a) * s->i_w + w * s_w + b) * s->i_c + ci];
            }
      }
  return 0;
}

/* Sub-matrix GEMM in the BLAS style of Sec. 2.1: A is the p x q
 * sub-matrix with top-left element *A and leading dimension lda; B is q x r
 * with leading dimension r; C is p x r with leading dimension ldc. */
static void gemm_submatrix(const double* A, int64_t lda, const double* B,
                           double* C, int64_t ldc, int64_t p, int64_t q,
                           int64_t r) {
  for (int64_t i = 0; i < p; ++i)
    for (int64_t j = 0; j < r; ++j) {
      double acc = 0.0;
      for (int64_t t = 0; t < q; ++t) acc += A[i * lda + t] * B[t * r + j];
      C[i * ldc + j] = acc;
    }
}

/* ------------------------------------------------------------ lowering */

/* Alg.2 l.3-6, P:155-159 (and Alg.1 l.4-6): for n, w, h in
 * 0:i_n x 0:o_w x 0:i_h, copy the k_w i_c contiguous elements of
 * I[n, h, s_w w : s_w w + k_w, 0:i_c] to L[n, w, h, 0:k_w, 0:i_c]. */
int mec_oracle_lower(const void* I, void* L, const mec_oracle_shape* s,
                     int s_h, int s_w, size_t elt) {
  int64_t oh, ow;
  if (!I || !L || elt == 0 || mec_oracle_out_dims(s, s_h, s_w, &oh, &ow)) return -1;
  const unsigned char* src = (const unsigned char*)I;
  unsigned char* dst = (unsigned char*)L;
  const int64_t strip = s->k_w * s->i_c; /* elements per copy */
  for (int64_t n = 0; n < s->i_n; ++n)
    for (int64_t w = 0; w < ow; ++w)
      for (int64_t h = 0; h < s->i_h; ++h) {
        int64_t l_off = (((n * ow + w) * s->i_h + h) * s->k_w) * s->i_c;
        int64_t i_off = ((n * s->i_h + h) * s->i_w + s_w * w) * s->i_c;
        memcpy(dst + (size_t)l_off * elt, src + (size_t)i_off * elt,
               (size_t)strip * elt);
      }
  return 0;
}

/* -------------------------------------------------------- Algorithm 1 */

/* Algorithm 1, with i_n = i_c = k_c = 1.  L is o_w x i_h x k_w,
 * then o_w x (i_h k_w); output row h is the sub-matrix
 * L[0:o_w, s_h k_w h : s_h k_w h + k_h k_w] times K (k_h k_w x 1), ld = i_h k_w
 * (P:100-102). */
int mec_oracle_vanilla_mec(const double* I, const double* K, double* O,
                           int64_t i_h, int64_t i_w, int64_t k_h, int64_t k_w,
                           int s_h, int s_w) {
  if (!I || !K || !O || i_h < k_h || i_w < k_w || k_h < 1 || k_w < 1 ||
      s_h < 1 || s_w < 1)
    return -1;
  const int64_t o_h = (i_h - k_h) / s_h + 1, o_w = (i_w - k_w) / s_w + 1;
  /* l.2: Allocate L with o_w i_h k_w elements */
  double* L = (double*)malloc(sizeof(double) * (size_t)(o_w * i_h * k_w));
  if (!L) return -3;
  /* l.4-6: L[w, h, 0:k_w] = I[h, s_w w : s_w w + k_w] */
  for (int64_t w = 0; w < o_w; ++w)
    for (int64_t h = 0; h < i_h; ++h)
      for (int64_t b = 0; b < k_w; ++b)
        L[(w * i_h + h) * k_w + b] = I[h * i_w + s_w * w + b];
  /* l.7-12: O[h, 0:o_w] = L[0:o_w, s_h k_w h : s_h k_w h + k_h k_w] x K */
  for (int64_t h = 0; h < o_h; ++h)
    gemm_submatrix(L + s_h * k_w * h, i_h * k_w, K, O + h * o_w, 1, o_w,
                   k_h * k_w, 1);
  free(L);
  return 0;
}

/* --------------------------------------------------------- Algorithm 2 */

static double* lower_double(const double* I, const mec_oracle_shape* s, int s_h,
                            int s_w) {
  int64_t nL = mec_oracle_elems_L_mec(s, s_h, s_w);
  double* L = (double*)malloc(sizeof(double) * (size_t)nL);
  if (!L) return NULL;
  mec_oracle_lower(I, L, s, s_h, s_w, sizeof(double));
  return L;
}

/* Solution A, Alg.2 l.9-19, literally. */
static int solA_on_L(double* L, const double* K, double* O,
                     const mec_oracle_shape* s, int s_h, int s_w) {
  int64_t o_h, o_w;
  mec_oracle_out_dims(s, s_h, s_w, &o_h, &o_w);
  const int64_t nO = mec_oracle_elems_O(s, s_h, s_w);
  const int64_t nL = mec_oracle_elems_L_mec(s, s_h, s_w);
  if (nO > nL) return -2; /* L must be at least as large as O */
  const int64_t row_len = s->i_h * s->k_w * s->i_c; /* l.9 ld of L */
  const int64_t kdim = s->k_h * s->k_w * s->i_c;
  const int64_t m = s->i_n * o_w;
  /* l.9: L as (i_n o_w) x (i_h k_w i_c); O as o_h x (i_n o_w k_c).
   * l.10-12: O[h, 0:i_n o_w k_c] = L[0:i_n o_w, s_h k_w i_c h : + k_h k_w i_c] x K */
  for (int64_t h = 0; h < o_h; ++h)
    gemm_submatrix(L + s_h * s->k_w * s->i_c * h, row_len, K,
                   O + h * m * s->k_c, s->k_c, m, kdim, s->k_c);
  /* l.13: Copy L = O */
  memcpy(L, O, sizeof(double) * (size_t)nO);
  /* l.14-19: L as o_h x i_n x (o_w k_c); O as i_n x o_h x (o_w k_c);
   * O[n, h, 0:o_w k_c] = L[h, n, 0:o_w k_c] */
  const int64_t blk = o_w * s->k_c;
  for (int64_t n = 0; n < s->i_n; ++n)
    for (int64_t h = 0; h < o_h; ++h)
      memcpy(O + (n * o_h + h) * blk, L + (h * s->i_n + n) * blk,
             sizeof(double) * (size_t)blk);
  return 0;
}

int mec_oracle_conv_solA(const double* I, const double* K, double* O,
                         const mec_oracle_shape* s, int s_h, int s_w) {
  if (!I || !K || !O || !shape_ok(s, s_h, s_w)) return -1;
  if (mec_oracle_elems_O(s, s_h, s_w) > mec_oracle_elems_L_mec(s, s_h, s_w))
    return -2;
  double* L = lower_double(I, s, s_h, s_w); /* l.2-6 */
  if (!L) return -3;
  int rc = solA_on_L(L, K, O, s, s_h, s_w);
  free(L);
  return rc;
}

typedef struct {
  const double *L, *K;
  double* O;
  const mec_oracle_shape* s;
  int s_h;
  int64_t o_h, o_w;
} solB_ctx;

/* Solution B, Alg.2 l.20-25: L as i_n matrices o_w x (i_h k_w i_c),
 * O as i_n matrices o_h x (o_w k_c);
 * O[n][h, 0:o_w k_c] = L[n][0:o_w, s_h k_w i_c h : + k_h k_w i_c] x K. */
static void solB_image(void* vctx, int64_t n) {
  const solB_ctx* c = (const solB_ctx*)vctx;
  const mec_oracle_shape* s = c->s;
  const int64_t row_len = s->i_h * s->k_w * s->i_c;
  const int64_t kdim = s->k_h * s->k_w * s->i_c;
  const double* Ln = c->L + n * c->o_w * row_len;
  double* On = c->O + n * c->o_h * c->o_w * s->k_c;
  for (int64_t h = 0; h < c->o_h; ++h)
    gemm_submatrix(Ln + c->s_h * s->k_w * s->i_c * h, row_len, c->K,
                   On + h * c->o_w * s->k_c, s->k_c, c->o_w, kdim, s->k_c);
}

static int solB_on_L(const double* L, const double* K, double* O,
                     const mec_oracle_shape* s, int s_h, int s_w, int n_threads) {
  solB_ctx c = {L, K, O, s, s_h, 0, 0};
  mec_oracle_out_dims(s, s_h, s_w, &c.o_h, &c.o_w);
  for_each_image(s->i_n, n_threads, solB_image, &c);
  return 0;
}

int mec_oracle_conv_solB(const double* I, const double* K, double* O,
                         const mec_oracle_shape* s, int s_h, int s_w,
                         int n_threads) {
  if (!I || !K || !O || !shape_ok(s, s_h, s_w)) return -1;
  double* L = lower_double(I, s, s_h, s_w); /* l.2-6 */
  if (!L) return -3;
  int rc = solB_on_L(L, K, O, s, s_h, s_w, n_threads);
  free(L);
  return rc;
}

/* Algorithm 2 end to end: l.1-6 lowering, l.7-8 the T test,
 * then Solution A (l.9-19) or Solution B (l.20-25). */
int mec_oracle_mec(const double* I, const double* K, double* O,
                   const mec_oracle_shape* s, int s_h, int s_w, int T,
                   int n_threads, int* path_out) {
  if (!I || !K || !O || !shape_ok(s, s_h, s_w)) return -1;
  int path = mec_oracle_select_path(s, s_h, s_w, T);
  if (path_out) *path_out = path;
  double* L = lower_double(I, s, s_h, s_w);
  if (!L) return -3;
  int rc = (path == 1) ? solA_on_L(L, K, O, s, s_h, s_w)
                       : solB_on_L(L, K, O, s, s_h, s_w, n_threads);
  free(L);
  return rc;
}
