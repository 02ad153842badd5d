/*
 * lowrank_b200.h -- C ABI of the B200-native ID / CUR hot path.
 *
 * Drop-in boundary for the reference library `lowrank` (header-only C++ on
 * Eigen, /root/reference/proj/include/lowrank).  Each entry point replaces
 * the reference template cited next to it; include/lowrank_b200/lowrank.hpp
 * re-declares the reference's C++ names (namespace lowrank) on top of this
 * ABI, and INTEGRATION.md shows the bindings.
 *
 * Conventions
 *   - matrices are column-major double with an explicit leading dimension;
 *     pivots are 0-based int64 (core.hpp:12-20);
 *   - outputs are caller-allocated;
 *   - plain names take HOST pointers (inputs copied to the GPU, outputs copied
 *     back, the call returns when results are on the host); the `_d`
 *     variants take DEVICE pointers and are stream-ordered on the context's
 *     stream (they still synchronise where the reference would throw, i.e.
 *     after validation reductions);
 *   - every call returns an LR_* status; the message of the last failure on
 *     the calling thread is lr_last_error(), mirroring the exception classes
 *     of core.hpp:22-42 (invalid_argument, SingularityError{index},
 *     ConvergenceError, runtime_error).
 *   - there is no CPU fallback: without a usable sm_100 device every call
 *     returns LR_ECUDA.
 */
#ifndef LOWRANK_B200_H
#define LOWRANK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define LR_OK 0
#define LR_EINVAL 1      /* std::invalid_argument                          */
#define LR_ESINGULAR 2   /* lowrank::SingularityError (lr_last_singular_index) */
#define LR_ECONVERGE 3   /* lowrank::ConvergenceError                      */
#define LR_ERUNTIME 4    /* std::runtime_error                             */
#define LR_ECUDA 5       /* device / driver failure                        */
#define LR_EUNSUPPORTED 6 /* reference feature not on the B200 path yet    */
#define LR_ENCCL 7        /* NCCL failure (column-sharded entry points)    */
#define LR_EPARSE 8       /* lowrank::ParseError (io.hpp readers)          */

/* SolveKind, solve.hpp:9 */
#define LR_SOLVE_BACKSUB 0
#define LR_SOLVE_PINV 1
#define LR_SOLVE_TIKHONOV 2

/* SketchKind, sketch.hpp:19 */
#define LR_SKETCH_GAUSSIAN 0
#define LR_SKETCH_SRFT 1

/* CUR middle factor */
#define LR_U_VT_RPINV 0       /* cur.hpp:30: u = col_basis()^T pinv(r)        */
#define LR_U_CPINV_A_RPINV 1  /* lowrank_main.cpp:215: u = pinv(c) a pinv(r)  */

/* SolveStrategy, solve.hpp:16-32 (defaults: BACKSUB, 1e-12, 0, escalate=1) */
typedef struct {
  int kind;
  double threshold;
  double ridge;
  int escalate;
} lr_solve_strategy;

/* SketchConfig, sketch.hpp:21-33 (defaults: GAUSSIAN, p=10, 0, q=0, 1, seed 0) */
typedef struct {
  int kind;
  int oversample;
  int64_t srft_samples;
  int power;
  int reorthonormalize;
  uint64_t seed;
} lr_sketch_config;

typedef struct lr_ctx lr_ctx;

typedef struct {
  long long cpqr_steps;      /* Householder steps run by the last call           */
  long long norm_recomputes; /* exact norm recomputations (cpqr.hpp:80-83)       */
  int solve_escalated;       /* 1 if the last coefficient solve took the pinv path */
  int pinv_fast_path;        /* 1 if the last CUR U used the CholeskyQR2 route    */
  int concurrent_tail;       /* 1 if the last CUR ran its row-ID and A^T Q_c chains
                                concurrently on two SM partitions (LRB_CUR_SPLIT)  */
} lr_stats;

lr_solve_strategy lr_solve_strategy_default(void);
lr_sketch_config lr_sketch_config_default(void);

const char* lr_last_error(void);
int64_t lr_last_singular_index(void);

int lr_ctx_create(lr_ctx** out, int device);
int lr_ctx_destroy(lr_ctx* ctx);
/* run subsequent _d calls on this cudaStream_t (NULL = the legacy default stream) */
int lr_ctx_set_stream(lr_ctx* ctx, void* cuda_stream);
/* engine for the two A-sized contractions (Y = Omega A, A^T Q):
   LR_GEMM_DMMA (default): FP64 tensor-core GEMM (DMMA), FP64 rounding per FMA;
   LR_GEMM_OZAKI_INT8: FP64 emulated on the INT8 tensor cores (Ozaki scheme II,
   16 moduli): exact integer products of the inputs truncated to 54+ bits
   relative to each column's largest entry (K <= 2^17; larger K uses DMMA).
   Power rounds (sketch.hpp:148-164) use it for both halves: A Y^T contracts
   over A's columns, so the column scales of A's cached residue planes are
   folded into Y^T and the planes enter the GEMM as the M-major operand. */
#define LR_GEMM_DMMA 0
#define LR_GEMM_OZAKI_INT8 1
int lr_ctx_set_gemm_mode(lr_ctx* ctx, int mode);
/* The device matrix a (m x n, lda) will be contracted more than once by the
   following calls (e.g. the column-sharded pipeline's sketch and A^T Q_c):
   on the Ozaki engine its residue planes are split once and reused until
   lr_ctx_clear_operand_cache.  The caller must not modify a in between. */
int lr_ctx_cache_operand(lr_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda);
int lr_ctx_clear_operand_cache(lr_ctx* ctx);
/* free the context's grow-only device workspace (Ozaki residue planes of A:
   2 bytes of HBM per byte of A, CPQR state, the call arena) */
int lr_ctx_release_workspace(lr_ctx* ctx);
int lr_ctx_get_gemm_mode(lr_ctx* ctx);
/* Schedule of the randomized CUR's tail (u_mode LR_U_CPINV_A_RPINV, large A).
   After C = A(:, J) two chains are independent: the row ID of C (CPQR of C^T,
   id.hpp:101-128) and Q_c -> A^T Q_c (lowrank_main.cpp:210-215).  sms > 0 runs
   them concurrently, the row ID on an SM partition of that size; 0 runs them
   one after the other; -1 (default) chooses: concurrent with 40 SMs (48 through the host-pointer entry, 56 for a tall A) when the
   INT8 engine contracts A, m, n >= 32768 and m n >= 2^31 (measured break-even).  Same kernels and index sets
   either way; the factors agree to roundoff (split-K depends on the SM count). */
int lr_ctx_set_concurrent_tail(lr_ctx* ctx, int sms);
/* back to the context's own (non-blocking) stream, the default after creation */
int lr_ctx_use_own_stream(lr_ctx* ctx);
int lr_ctx_get_stats(lr_ctx* ctx, lr_stats* out);
int lr_ctx_synchronize(lr_ctx* ctx);
/* per-stage device time with CUDA events on the context stream (tracing):
   enable, then read a JSON object {stage: {ms, count}} accumulated since the
   last reset (the report synchronises the stream) */
int lr_ctx_enable_timing(lr_ctx* ctx, int on);
int lr_ctx_stage_report(lr_ctx* ctx, char* buf, int64_t buflen);
int lr_ctx_reset_stats(lr_ctx* ctx);
/* number of kernels this library has launched in the process */
long long lr_kernel_launches(void);

/* rng.hpp:74-94 gaussian_matrix<double>(rows, cols, seed): out rows x cols (ld rows) */
int lr_gaussian_matrix(lr_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out);
int lr_gaussian_matrix_d(lr_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out, int64_t ldo);

/* sketch.hpp:67-78 sketch_gaussian(a, ell, seed).y: y ell x n (ld ell) */
int lr_sketch_gaussian(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell,
                       uint64_t seed, double* y);
int lr_sketch_gaussian_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell,
                         uint64_t seed, double* y, int64_t ldy);
/* sketch.hpp:84-100 srft_operator: out (ell x m, ld ell) */
int lr_srft_operator(lr_ctx* ctx, int64_t m, int64_t ell, uint64_t seed, double* out);
/* svd.hpp:216-235 orth_rows: thin Q^T of the Householder QR of y^T, rank-trimmed:
   out (ell x n, ld ell; first *r rows) */
int lr_orth_rows(lr_ctx* ctx, int64_t ell, int64_t n, const double* y, int64_t ldy, double* out, int64_t* r);
/* sketch.hpp:238-254 randomized_svd: u (m x k), sigma (k), v (n x k) */
int lr_randomized_svd(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                      lr_sketch_config cfg, double* u, double* sigma, double* v);
/* sketch.hpp:84-143 sketch_srft: y (ell x n, ld ell) = sqrt(m/ell) R H D A (random
   signs D, orthonormal Hartley transform H, ell sampled rows R) */
int lr_sketch_srft(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, uint64_t seed,
                   double* y);
/* sketch.hpp:148-164 sketch_power: y (ell x n, ld ell) = Omega A (A^T A)^q with
   optional row re-orthonormalisation (svd.hpp:216-235); *rows = final row
   count (orth_rows drops numerically dependent rows) */
int lr_sketch_power(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, int q,
                    int reorth, uint64_t seed, double* y, int64_t* rows);

/* cpqr.hpp:32-114 cpqr_partial(a, k): q m x k (may be NULL), s k x n, pivots n */
int lr_cpqr_partial(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, double* q,
                    double* s, int64_t* pivots);
int lr_cpqr_partial_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, double* q,
                      double* s, int64_t* pivots);
/* cpqr.hpp:118-122 cpqr_full(a): k = min(m, n) */
int lr_cpqr_full(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, double* q, double* s,
                 int64_t* pivots);

/* solve.hpp:104-145 stabilized_coeff_solve(s11, s12, strategy): t k x nc */
int lr_stabilized_coeff_solve(lr_ctx* ctx, int64_t k, int64_t nc, const double* s11, int64_t ld11,
                              const double* s12, int64_t ld12, lr_solve_strategy strategy, double* t);

/* svd.hpp:132-183 svd(a): r = min(m,n); u m x r, sigma r, v n x r */
int lr_svd(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, double* u, double* sigma, double* v);
/* svd.hpp:193-207 pinv(a, threshold): out n x m */
int lr_pinv(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, double threshold, double* out);

/* id.hpp:91-105 id_column(a, k, strategy): pivots n, coeff k x (n-k) */
int lr_id_column(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                 lr_solve_strategy strategy, int64_t* pivots, double* coeff);
int lr_id_column_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                   lr_solve_strategy strategy, int64_t* pivots, double* coeff);
/* id.hpp:108-119 id_row(a, k, strategy): pivots m, coeff k x (m-k) */
int lr_id_row(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
              lr_solve_strategy strategy, int64_t* pivots, double* coeff);

/* sketch.hpp:200-223 randomized_id(a, k, cfg, strategy): pivots n, coeff k x (n-k) */
int lr_randomized_id(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                     lr_sketch_config cfg, lr_solve_strategy strategy, int64_t* pivots, double* coeff);
int lr_randomized_id_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                       lr_sketch_config cfg, lr_solve_strategy strategy, int64_t* pivots, double* coeff);

/* id.hpp:124-134 tsid_from_column_id(a, col_id, strategy): row pivots m,
   row coeff k x (m-k), skeleton k x k.  (col coeff is carried by the caller) */
int lr_tsid_from_column_id(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                           const int64_t* col_pivots, lr_solve_strategy strategy, int64_t* row_pivots,
                           double* row_coeff, double* skeleton);

/* cur.hpp:23-34 cur_from_two_sided(a, tsid, thr) (u_mode LR_U_VT_RPINV) or the
   lowrank_main.cpp:215 middle factor (LR_U_CPINV_A_RPINV): c m x k, u k x k, r k x n */
int lr_cur_from_two_sided(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                          const int64_t* col_pivots, const double* col_coeff, const int64_t* row_pivots,
                          double pinv_threshold, int u_mode, double* c, double* u, double* r);

/* sketch.hpp:227-234 randomized_cur(a, k, cfg, strategy, thr) (+ u_mode).
   Optional outputs (may be NULL): col_coeff k x (n-k), row_coeff k x (m-k), skeleton k x k */
int lr_randomized_cur(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                      lr_sketch_config cfg, lr_solve_strategy strategy, double pinv_threshold, int u_mode,
                      int64_t* col_pivots, int64_t* row_pivots, double* c, double* u, double* r,
                      double* col_coeff, double* row_coeff, double* skeleton);
int lr_randomized_cur_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                        lr_sketch_config cfg, lr_solve_strategy strategy, double pinv_threshold, int u_mode,
                        int64_t* col_pivots, int64_t* row_pivots, double* c, double* u, double* r,
                        double* col_coeff, double* row_coeff, double* skeleton);

/* cur.hpp:37-42 cur_id(a, k, strategy, thr) (+ u_mode), deterministic */
int lr_cur_id(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
              lr_solve_strategy strategy, double pinv_threshold, int u_mode, int64_t* col_pivots,
              int64_t* row_pivots, double* c, double* u, double* r, double* col_coeff, double* row_coeff,
              double* skeleton);
int lr_cur_id_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                lr_solve_strategy strategy, double pinv_threshold, int u_mode, int64_t* col_pivots,
                int64_t* row_pivots, double* c, double* u, double* r, double* col_coeff, double* row_coeff,
                double* skeleton);

/* ||A - C U R||_F and ||A||_F (core.hpp:64-67 on cur.hpp:77-80): out[0], out[1] */
int lr_cur_error_fro(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                     const double* c, const double* u, const double* r, double* out);
int lr_cur_error_fro_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                       const double* c, const double* u, const double* r, double* out);

/* ---- BASELINE config 5: randomized CUR of a CSR matrix (device pointers,
   int64 indices).  The reference is dense-only (core.hpp:14-17); these apply
   sketch.hpp:227-234 (+ lowrank_main.cpp:215 when u_mode says so) to the
   densified matrix, with C = A(:, J) returned as a CSC extract and R = A(I, :)
   as a CSR extract (index/value buffers need capacity nnz; the used length is
   c_col_ptr[k] / r_row_ptr[k]).  col_coeff, row_coeff, skeleton may be NULL. */
int lr_randomized_cur_csr_d(lr_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                            const int64_t* col_idx, const double* val, int64_t k, lr_sketch_config cfg,
                            lr_solve_strategy strategy, double pinv_threshold, int u_mode, int64_t* col_pivots,
                            int64_t* row_pivots, double* u, int64_t* c_col_ptr, int64_t* c_row_idx, double* c_val,
                            int64_t* r_row_ptr, int64_t* r_col_idx, double* r_val, double* col_coeff,
                            double* row_coeff, double* skeleton);
/* ||A - C U R||_F, ||A||_F for the sparse factors above: out[0], out[1] */
int lr_cur_error_fro_csr_d(lr_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                           const int64_t* col_idx, const double* val, int64_t k, const int64_t* c_col_ptr,
                           const int64_t* c_row_idx, const double* c_val, const double* u,
                           const int64_t* r_row_ptr, const int64_t* r_col_idx, const double* r_val, double* out);

/* ---- shard-level primitives (device pointers) used by the column-sharded
   multi-GPU orchestration (paper_1412_8447_b200/distributed.py) ---- */
/* sketch.hpp:210-221: CPQR of a sample y (ell x n) then the coefficient solve */
int lr_id_from_sample_d(lr_ctx* ctx, int64_t ell, int64_t n, const double* y, int64_t ldy, int64_t k,
                        lr_solve_strategy strategy, int64_t* pivots, double* coeff);
/* id.hpp:124-134 given the column skeleton c = A(:, J) (m x k) */
int lr_tsid_from_skeleton_columns_d(lr_ctx* ctx, int64_t m, int64_t k, const double* c, int64_t ldc,
                                    lr_solve_strategy strategy, int64_t* row_pivots, double* row_coeff,
                                    double* skeleton);
/* core.hpp:70-85 gathers; a negative column index gathers a zero column */
int lr_gather_columns_d(lr_ctx* ctx, int64_t m, int64_t k, const double* a, int64_t lda, const int64_t* idx,
                        double* out, int64_t ldo);
int lr_gather_rows_d(lr_ctx* ctx, int64_t k, int64_t n, const double* a, int64_t lda, const int64_t* idx,
                     double* out, int64_t ldo);
int lr_transpose_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, double* out, int64_t ldo);
int lr_cholesky_upper_d(lr_ctx* ctx, int64_t k, double* g, int64_t ldg);
int lr_tri_upper_inverse_d(lr_ctx* ctx, int64_t k, const double* r, int64_t ldr, double* rinv, int64_t ldi);
int lr_cholqr2_d(lr_ctx* ctx, int64_t rows, int64_t k, const double* x, int64_t ldx, double* r, double* rinv,
                 int* ok);

/* C (m x n) = A (m x k) B (k x n) on the GPU (FP64 DMMA): the products of the
   reconstructions id.hpp:143-159 / cur.hpp:77-80; host and device pointers */
int lr_gemm(lr_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, const double* b,
            int64_t ldb, double* c, int64_t ldc);
int lr_gemm_d(lr_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, const double* b,
              int64_t ldb, double* c, int64_t ldc);
/* Y (M x N) = P^T Q on the context's contraction engine (benchmark / test access) */
int lr_gemm_tn_d(lr_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* P, int64_t ldp, const double* Q,
                 int64_t ldq, double* out, int64_t ldo);

/* ---- column-sharded multi-GPU entry points (one process per GPU; SURVEY.md
   section 8e).  Rank g passes its column block A(:, col_offset : col_offset +
   n_local) of the m x n_total matrix (device pointer).  The CPQRs run sharded:
   per step one ncclAllGather carries every rank's pivot candidate (norm^2,
   logical position, the column), every rank applies the winner's reflector to
   its own columns (cpqr.hpp:48-85) -- no rank holds the whole sample.  Outputs
   are replicated on every rank except R, of which each rank gets its column
   block (k x n_local).  Without an attached communicator the same code runs
   for one unsharded rank (col_offset 0, n_local = n_total).  The reference's
   interface has no multi-process form; these extend lr_randomized_cur_d
   (sketch.hpp:227-234, lowrank_main.cpp:215) and lr_cpqr_partial_d
   (cpqr.hpp:32-114). ---- */
/* NCCL unique id (128 bytes) made on one rank and shared with the others */
int lr_nccl_get_unique_id(unsigned char* id);
/* bind an NCCL communicator (ncclCommInitRank over the process's libnccl.so.2) */
int lr_ctx_attach_comm(lr_ctx* ctx, const unsigned char* id, int nranks, int rank);
int lr_ctx_detach_comm(lr_ctx* ctx);
int lr_ctx_comm_info(lr_ctx* ctx, int* nranks, int* rank);
/* test vehicle: without a communicator, run the sharded CPQRs as `nshards`
   column blocks inside this process (each step: the blocks' candidates are
   gathered by device copies, then every block's step kernel runs; no kernel
   waits on another).  0 = off. */
int lr_ctx_set_shard_emulation(lr_ctx* ctx, int nshards);
/* pivots (n_total) and the sign-fixed top k rows of R in logical column order
   (s, k x n_total, ld k), replicated */
int lr_cpqr_sharded_d(lr_ctx* ctx, int64_t m, int64_t n_local, int64_t col_offset, int64_t n_total,
                      const double* a_local, int64_t lda, int64_t k, int64_t* pivots, double* s);
/* host pointers: the rank's block is uploaded in column chunks with the sketch
   of each chunk overlapped with the transfer; outputs back in host memory */
int lr_randomized_cur_sharded(lr_ctx* ctx, int64_t m, int64_t n_local, int64_t col_offset, int64_t n_total,
                              const double* a_local, int64_t lda, int64_t k, lr_sketch_config cfg,
                              lr_solve_strategy strategy, double pinv_threshold, int u_mode, int64_t* col_pivots,
                              int64_t* row_pivots, double* c, double* u, double* r_local, double* col_coeff,
                              double* row_coeff, double* skeleton);
/* randomized CUR (Gaussian sketch, q = 0) of the column-sharded A; u_mode as
   lr_randomized_cur_d; r_local is this rank's k x n_local block of R */
int lr_randomized_cur_sharded_d(lr_ctx* ctx, int64_t m, int64_t n_local, int64_t col_offset, int64_t n_total,
                                const double* a_local, int64_t lda, int64_t k, lr_sketch_config cfg,
                                lr_solve_strategy strategy, double pinv_threshold, int u_mode,
                                int64_t* col_pivots, int64_t* row_pivots, double* c, double* u, double* r_local,
                                double* col_coeff, double* row_coeff, double* skeleton);

/* ---- the reference's binary matrix format (io.hpp:197-233: two little-endian
   int64 dimensions, then row-major doubles) straight to / from device memory:
   the file streams through page-locked buffers in row blocks, each block is
   copied to the GPU while the next is read, and transposed there into the
   column-major layout every entry point takes.  Errors follow io.hpp
   (LR_EPARSE + the reference's messages). ---- */
/* out == NULL: only *rows / *cols are read (size the buffer); else out is
   rows x cols column-major with leading dimension ldo */
int lr_read_matrix_binary_d(lr_ctx* ctx, const char* path, int64_t* rows, int64_t* cols, double* out, int64_t ldo);
int lr_write_matrix_binary_d(lr_ctx* ctx, const char* path, int64_t m, int64_t n, const double* a, int64_t lda);

/* ---- verifiers at scale (verify.hpp:14-166).  The reference takes every
   spectral norm as sigma_1 of a full SVD of the materialised m x n residual
   (svd.hpp:185-189); here the residual A - X Y stays an operator and sigma_1
   comes from a seeded block Krylov iteration on E^T E (converged to 1e-14
   relative, from below); Frobenius norms by the fused residual GEMM. ---- */
typedef struct lr_error_report { /* verify.hpp:22-28 */
  double abs_spectral, rel_spectral, abs_frob, rel_frob;
  int rel_is_absolute;
} lr_error_report;
typedef struct lr_lemma1_report { /* verify.hpp:60-66 */
  double lhs, rhs, e_norm, etilde_norm;
  int holds;
} lr_lemma1_report;
typedef struct lr_lemma2_report { /* verify.hpp:86-95 */
  double etilde_norm, fe_norm, entry_diff, e_norm, t_norm, bound_rhs;
  int holds, bound_holds;
} lr_lemma2_report;
typedef struct lr_corollary_report { /* verify.hpp:136-143 */
  double lhs, bound, t_norm, e_norm, ceiling;
  int holds;
} lr_corollary_report;
/* ||A - X Y||_2 and ||A - X Y||_F (X m x k, Y k x n; k = 0: of A); either output may be NULL */
int lr_residual_norms_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                        const double* x, int64_t ldx, const double* y, int64_t ldy, double* spectral,
                        double* frobenius);
/* verify.hpp:31-56 error_report(a, approx) for approx = X Y */
int lr_error_report_lowrank_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                              const double* x, int64_t ldx, const double* y, int64_t ldy, lr_error_report* out);
/* verify.hpp:70-80 verify_lemma1(a, cur, col_id, row_basis): the CUR given by its
   index sets, coefficient blocks and U (C, R, W rebuilt from A) */
int lr_verify_lemma1_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                       const int64_t* col_pivots, const double* col_coeff, const int64_t* row_pivots,
                       const double* row_coeff, const double* u, lr_lemma1_report* out);
/* verify.hpp:97-130 verify_lemma2(a, col_id, row_id) */
int lr_verify_lemma2_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                       const int64_t* col_pivots, const double* col_coeff, const int64_t* row_pivots,
                       const double* row_coeff, lr_lemma2_report* out);
/* verify.hpp:144-160 verify_corollary(a, cur, col_id, strategy) */
int lr_verify_corollary_d(lr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                          const int64_t* col_pivots, const double* col_coeff, const double* u,
                          lr_solve_strategy strategy, lr_corollary_report* out);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif
