/*
 * mec_oracle.h -- plain, slow, obviously-correct CPU oracle for MEC
 * (Cho & Brand, "MEC: Memory-efficient Convolution for Deep Neural Network",
 * ICML 2017, arXiv 1706.06873; cited below as P:<line> of PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1706_06873_b200/csrc) and neither side includes the other.
 *
 * Conventions (Table 1; Sec. 2.1):
 *   I : i_n x i_h x i_w x i_c   (n-h-w-c, row-major, zero padding pre-applied)
 *   K : k_h x k_w x i_c x k_c   (read as a (k_h k_w i_c) x k_c matrix, Alg.2 l.7)
 *   O : i_n x o_h x o_w x k_c   (n-h-w-c)
 *   L : i_n x o_w x i_h x k_w x i_c
 * All floating-point arithmetic is double precision.
 */
#ifndef MEC_ORACLE_H
#define MEC_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t i_n, i_h, i_w, i_c, k_h, k_w, k_c;
} mec_oracle_shape;

/* Eq. (1): o = (i - k) / s + 1, integer floor (reading Q1).
 * Returns 0 on success, -1 if i < k or s < 1 or any extent < 1. */
int mec_oracle_out_dims(const mec_oracle_shape* s, int s_h, int s_w,
                        int64_t* o_h, int64_t* o_w);

/* Element counts.  #L_MEC (Table 1 L dims P:27, Alg.2 l.2 P:154), #L_im2col
 * (Eq. 2, with i_c for the printed k_c: reading Q2), #O (Alg.2 l.1). */
int64_t mec_oracle_elems_L_mec(const mec_oracle_shape* s, int s_h, int s_w);
int64_t mec_oracle_elems_L_im2col(const mec_oracle_shape* s, int s_h, int s_w);
int64_t mec_oracle_elems_O(const mec_oracle_shape* s, int s_h, int s_w);

/* Alg.2 l.8: returns 1 (Solution A) iff o_w <= T and
 * #O <= #L, else 2 (Solution B). -1 on invalid shape. */
int mec_oracle_select_path(const mec_oracle_shape* s, int s_h, int s_w, int T);

/* Direct convolution (Fig. 1(a)): O[n,h,w,c] =
 *   sum_{a<k_h, b<k_w, ci<i_c} I[n, h s_h + a, w s_w + b, ci] * K[a,b,ci,c].
 * Threads split the images (n) only; each output is one plain double sum. */
int mec_oracle_direct_conv(const double* I, const double* K, double* O,
                           const mec_oracle_shape* s, int s_h, int s_w,
                           int n_threads);

/* im2col lowering (Fig. 1(b)): C is (i_n o_h o_w) x (k_h k_w i_c),
 * row (n,h,w), column (a,b,ci) -> I[n, h s_h + a, w s_w + b, ci]. */
int mec_oracle_im2col(const double* I, double* C, const mec_oracle_shape* s,
                      int s_h, int s_w);

/* MEC compact lowering, Alg.2 l.3-6:
 *   L[n,w,h,0:k_w,0:i_c] = I[n,h,s_w w : s_w w + k_w, 0:i_c]
 * for n < i_n, w < o_w, h < i_h (all input rows: reading Q5).
 * A pure element copy of elt_bytes-sized elements (bit-exact reference). */
int mec_oracle_lower(const void* I, void* L, const mec_oracle_shape* s,
                     int s_h, int s_w, size_t elt_bytes);

/* Algorithm 1, VanillaMEC, i_n = i_c = k_c = 1:
 * I is i_h x i_w, K is k_h x k_w, O is o_h x o_w. */
int mec_oracle_vanilla_mec(const double* I, const double* K, double* O,
                           int64_t i_h, int64_t i_w, int64_t k_h, int64_t k_w,
                           int s_h, int s_w);

/* Algorithm 2 Solution A (l.9-19), literal:
 * o_h GEMMs of (i_n o_w) x (k_h k_w i_c) windows of L times K into O in
 * h-n-w-c, "Copy L = O", then O[n,h,:] = L[h,n,:].
 * Returns -2 if #O > #L (Solution A unavailable). */
int mec_oracle_conv_solA(const double* I, const double* K, double* O,
                         const mec_oracle_shape* s, int s_h, int s_w);

/* Algorithm 2 Solution B (l.20-25): i_n o_h GEMMs of
 * o_w x (k_h k_w i_c) windows of L[n] times K, written directly in n-h-w-c.
 * Threads split the images (n) only. */
int mec_oracle_conv_solB(const double* I, const double* K, double* O,
                         const mec_oracle_shape* s, int s_h, int s_w,
                         int n_threads);

/* Algorithm 2 as written: lowering, then the l.8 test with threshold T picks
 * Solution A or B.  *path_out receives 1 (A) or 2 (B). */
int mec_oracle_mec(const double* I, const double* K, double* O,
                   const mec_oracle_shape* s, int s_h, int s_w, int T,
                   int n_threads, int* path_out);

#ifdef __cplusplus
}
#endif
#endif
