/*
 * lowrank_oracle.h -- CPU restatement of the reference ID / CUR hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 product path (paper_1412_8447_b200/csrc).  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product path never links it and never
 * falls back to it.
 *
 * Every routine restates the behaviour of the reference headers under
 * /root/reference/proj/include/lowrank (cited per function as file:line).
 * Parity pin: the restatement is checked against the reference's own
 * headers compiled in place (oracle/_ref, see oracle/Makefile and
 * oracle/eigen_subset/) on seeded inputs, and against the known-answer /
 * property cases of proj/tests/ (*.cpp) (tests/test_oracle.py).
 *
 * Storage is column-major double with explicit leading dimensions; pivots
 * are 0-based int64 (core.hpp:12-20).
 */
#ifndef LOWRANK_ORACLE_H
#define LOWRANK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mirror the exception classes of core.hpp:22-42) */
#define LRO_OK 0
#define LRO_EINVAL 1     /* std::invalid_argument */
#define LRO_ESINGULAR 2  /* lowrank::SingularityError (index reported) */
#define LRO_ECONVERGE 3  /* lowrank::ConvergenceError */
#define LRO_ERUNTIME 4   /* std::runtime_error */
#define LRO_ENOMEM 5

/* SolveKind (solve.hpp:9) */
#define LRO_SOLVE_BACKSUB 0
#define LRO_SOLVE_PINV 1
#define LRO_SOLVE_TIKHONOV 2

/* CUR middle-factor forms */
#define LRO_U_VT_RPINV 0      /* cur.hpp:30  u = basis()^T pinv(r) */
#define LRO_U_CPINV_A_RPINV 1 /* lowrank_main.cpp:215  u = pinv(c) a pinv(r) */

typedef struct {
  int kind;          /* LRO_SOLVE_* */
  double threshold;  /* default 1e-12 */
  double ridge;      /* Tikhonov weight */
  int escalate;      /* default 1 */
} lro_solve_strategy;

const char* lro_last_error(void);
int64_t lro_last_singular_index(void);
void lro_set_threads(int n); /* OpenMP threads for the GEMM helpers (0 = all) */

/* rng.hpp:14-34 */
uint64_t lro_mix64(uint64_t z);
uint64_t lro_stream_value(uint64_t seed, uint64_t index);
uint64_t lro_derive_seed(uint64_t seed, uint64_t tag);
/* rng.hpp:74-94: rows x cols, column-major, ld = rows */
int lro_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out);

/* C(MxN) = A(MxK) B(KxN), column-major, per-element sum over k ascending */
void lro_gemm_nn(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                 const double* B, int64_t ldb, double* C, int64_t ldc);

/* cpqr.hpp:32-114.  s is k x n (ld k); q (m x k, ld m) may be NULL;
 * tau (k) may be NULL; stats[0] <- number of exact norm recomputes. */
int lro_cpqr(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
             double* q, double* s, int64_t* pivots, double* tau, int64_t* stats);

/* solve.hpp:104-145.  t is k x nc (ld k). */
int lro_coeff_solve(int64_t k, int64_t nc, const double* s11, int64_t ld11,
                    const double* s12, int64_t ld12, lro_solve_strategy strat,
                    double* t);

/* svd.hpp:132-183: thin SVD, r = min(m,n); u m x r, sigma r, v n x r */
int lro_svd(int64_t m, int64_t n, const double* a, int64_t lda, double* u,
            double* sigma, double* v);
/* svd.hpp:193-207: out is n x m */
int lro_pinv(int64_t m, int64_t n, const double* a, int64_t lda, double threshold,
             double* out);

/* id.hpp:91-105: pivots n, coeff k x (n-k) */
int lro_id_column(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                  lro_solve_strategy strat, int64_t* pivots, double* coeff);
/* id.hpp:108-119: pivots m, coeff k x (m-k) */
int lro_id_row(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
               lro_solve_strategy strat, int64_t* pivots, double* coeff);

/* sketch.hpp:67-78: y is ell x n */
int lro_sketch_gaussian(int64_t m, int64_t n, const double* a, int64_t lda,
                        int64_t ell, uint64_t seed, double* y);
/* sketch.hpp:200-223 (Gaussian sketch, power q = 0): pivots n, coeff k x (n-k) */
int lro_randomized_id(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                      int oversample, uint64_t seed, lro_solve_strategy strat,
                      int64_t* pivots, double* coeff, int64_t* stats);

/* rng.hpp:53-62 CounterRng::sample_without_replacement (partial Fisher-Yates):
 * out[0..count) */
void lro_sample_without_replacement(uint64_t seed, int64_t population, int64_t count, int64_t* out);
/* sketch.hpp:84-100 srft_operator: ell x m dense operator, ld ell */
int lro_srft_operator(int64_t m, int64_t ell, uint64_t seed, double* out);
/* sketch.hpp:110-143 sketch_srft: y (ell x n, ld ell); radix-2 fast Hartley
 * transform (hartley.hpp:17-43) when m is a power of two, else the dense operator */
int lro_sketch_srft(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, uint64_t seed, double* y);
/* sketch.hpp:167-223 randomized_id with a full SketchConfig: kind 0 Gaussian / 1
 * SRFT, sample count k + oversample (Gaussian) or srft_samples (0 -> 2k), q power rounds */
int lro_randomized_id_cfg(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int kind, int oversample,
                          int64_t srft_samples, int q, int reorth, uint64_t seed, lro_solve_strategy strat,
                          int64_t* pivots, double* coeff, int64_t* stats);

/* sketch.hpp:238-254 randomized_svd: u m x k, sigma k, v n x k (kind/oversample/
 * srft_samples/q/reorth/seed as lro_randomized_id_cfg) */
int lro_randomized_svd(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int kind, int oversample,
                       int64_t srft_samples, int q, int reorth, uint64_t seed, double* u, double* sigma, double* v);

/* svd.hpp:216-235 orth_rows: Householder QR of y^T (n x ell), numerical rank
 * r (trailing |R_ii| <= max|R_ii| eps max(n, ell) dropped), out = thin Q^T:
 * r x n (ld ell; rows r..ell-1 untouched); *r_out = r */
int lro_orth_rows(int64_t ell, int64_t n, const double* y, int64_t ldy, double* out, int64_t* r_out);
/* sketch.hpp:148-164 sketch_power: y (ell x n, ld ell) = Omega A (A^T A)^q,
 * optional re-orthonormalisation; *rows_out = the sample's final row count */
int lro_sketch_power(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, int q, int reorth,
                     uint64_t seed, double* y, int64_t* rows_out);
/* sketch.hpp:200-223 with the Gaussian power sketch (q >= 0) */
int lro_randomized_id_power(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int oversample,
                            int q, int reorth, uint64_t seed, lro_solve_strategy strat, int64_t* pivots,
                            double* coeff, int64_t* stats);

/* id.hpp:124-134 given col pivots (n) and k: row pivots (m), row coeff
 * k x (m-k), skeleton k x k */
int lro_tsid_from_column_id(int64_t m, int64_t n, const double* a, int64_t lda,
                            int64_t k, const int64_t* col_pivots,
                            lro_solve_strategy strat, int64_t* row_pivots,
                            double* row_coeff, double* skeleton);

/* cur.hpp:23-34 (u_mode 0) / lowrank_main.cpp:210-215 (u_mode 1):
 * c m x k, u k x k, r k x n */
int lro_cur_from_two_sided(int64_t m, int64_t n, const double* a, int64_t lda,
                           int64_t k, const int64_t* col_pivots,
                           const double* col_coeff, const int64_t* row_pivots,
                           double pinv_threshold, int u_mode, double* c, double* u,
                           double* r);

/* ||A - C U R||_F (core.hpp:64-67 on the cur.hpp:77-80 reconstruction);
 * returns abs error and ||A||_F through out[0], out[1]. */
int lro_cur_error_fro(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                      const double* c, const double* u, const double* r, double* out);

#ifdef __cplusplus
}
#endif

#endif
