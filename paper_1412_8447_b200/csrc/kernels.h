// kernels.h -- host-side entry points of the device kernels (internal to the
// library; the public boundary is include/lowrank_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

namespace lrb {

enum { kEpiStore = 0, kEpiSplitK = 1, kEpiResid = 2 };

// Named, grow-only device scratch buffers owned by a context.
enum class WsSlot : int {
  kSplitK = 0,
  kOmega,
  kSample,
  kWork,
  kCpqrState,
  kCand,
  kTri,
  kTri2,
  kTmp0,
  kTmp1,
  kTmp2,
  kTmp3,
  kTmp4,
  kTmp5,
  kTmp6,
  kTmp7,
  kPartials,
  kHostCopyA,
  kHostCopyB,
  kOzA,        // Ozaki residue planes of the input matrix (kept across calls: no pool churn)
  kOzAShift,
  kOzP,        // residue planes of the other operand(s) of a contraction
  kOzPShift,
  kOzQ,
  kOzQShift,
  kShard,      // sharded CPQR state (shard.cu)
  kCount
};

class Workspace {
 public:
  Workspace() : ptr_((size_t)WsSlot::kCount, nullptr), cap_((size_t)WsSlot::kCount, 0) {}
  ~Workspace();
  void* get(WsSlot s, size_t bytes);
  // like get(), but nullptr instead of an exception when the device is out of memory
  void* try_get(WsSlot s, size_t bytes);
  double* get_doubles(WsSlot s, size_t n) { return static_cast<double*>(get(s, n * sizeof(double))); }
  void release_all();
  void swap(Workspace& o) noexcept {
    ptr_.swap(o.ptr_);
    cap_.swap(o.cap_);
  }
  Workspace(const Workspace&) = delete;  // owns device allocations
  Workspace& operator=(const Workspace&) = delete;

 private:
  std::vector<void*> ptr_;
  std::vector<size_t> cap_;
};

// ---------------------------------------------------------------- GEMM
int gemm_tn_grid_ctas(int M, int N);
// out(MxN) = alpha P^T Q + beta out; P: KxM (ldp), Q: KxN (ldq), K-contiguous.
// splits <= 0 chooses a deterministic split-K factor from the shape.  upper:
// only the output tiles on/above the diagonal (Gram products, M == N; the
// strictly-lower tiles are left unwritten).
void gemm_tn(Workspace& ws, int M, int N, int K, const double* P, int64_t ldp, const double* Q, int64_t ldq,
             double* out, int64_t ldo, double alpha, double beta, int splits, cudaStream_t st, bool upper = false,
             int tri = 0);
// tri bits for gemm_tn: the K-tiles that only meet structural zeros are skipped
constexpr int kTriP = 1;  // P(k, i) = 0 for k < i (P = U^T of an upper-triangular U: out = U Q)
constexpr int kTriQ = 2;  // Q(k, j) = 0 for k > j (Q upper triangular: out = P^T Q)
// per-CTA partial sums of (R - P^T Q)^2 written to partials_out[0..*num_partials)
void gemm_tn_resid_sq(Workspace& ws, int M, int N, int K, const double* P, int64_t ldp, const double* Q,
                      int64_t ldq, const double* R, int64_t ldr, double* partials_out, int* num_partials,
                      cudaStream_t st);

// ---------------------------------------------------------------- rng
// rows x cols Gaussian matrix with the reference stream semantics.  If
// transposed, writes out^T (cols x rows, ld = ldo) instead.
void gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out, int64_t ldo, bool transposed,
                     cudaStream_t st);

// sketch.hpp:84-100 SRFT operator transposed (m x ell, ld ldo) for sampled rows `rows` (device, ell)
void srft_operator_t(int64_t m, int64_t ell, uint64_t sign_seed, const int64_t* rows, double* out, int64_t ldo,
                     cudaStream_t st);

// ---------------------------------------------------------------- elementwise / data movement
void scale_matrix(int M, int N, double* a, int64_t lda, double beta, cudaStream_t st);
void copy_matrix(int64_t m, int64_t n, const double* src, int64_t lds, double* dst, int64_t ldd, cudaStream_t st);
// dst (k x k) = upper triangle of src, strict lower part zero
void copy_upper(int64_t k, const double* src, int64_t lds, double* dst, int64_t ldd, cudaStream_t st);
void transpose_matrix(int64_t m, int64_t n, const double* src, int64_t lds, double* dst, int64_t ldd,
                      cudaStream_t st);
void gather_columns(int64_t m, int64_t k, const double* a, int64_t lda, const int64_t* idx, double* out,
                    int64_t ldo, cudaStream_t st);
// out(i, j) = a(idx[i], j): k x n (ldo)
void gather_rows(int64_t k, int64_t n, const double* a, int64_t lda, const int64_t* idx, double* out,
                 int64_t ldo, cudaStream_t st);
// out(j, i) = a(idx[i], j): n x k (ldo), i.e. the transpose of gather_rows
void gather_rows_t(int64_t k, int64_t n, const double* a, int64_t lda, const int64_t* idx, double* out,
                   int64_t ldo, cudaStream_t st);
// flag[0] |= 1 if any entry non-finite
void check_finite(int64_t m, int64_t n, const double* a, int64_t lda, int* flag, cudaStream_t st);
// deterministic sum of n doubles into out[0] (single block, fixed order)
void sum_partials(const double* p, int n, double* out, cudaStream_t st);
// per-column squared norms summed: partial sums of squares of a (m x n) -> out[0]
void frob2(int64_t m, int64_t n, const double* a, int64_t lda, double* partials, double* out, cudaStream_t st);

// ---------------------------------------------------------------- CPQR
struct CpqrStats {
  long long recomputes;
};
// Truncated column-pivoted Householder QR (cpqr.hpp:32-114) of W (m x n,
// ld), in place: after return the upper part holds s (unsigned), the strict
// lower part the reflectors, pivots the permutation and tau the k scalars.
// Device pointers; pivots (n int64), tau (k), flags (1 int: nonfinite input).
// `padded`: ld % 64 == 0 and rows [m, ld) of W are zero (enables the fast path).
// nopivot: unpivoted Householder QR with the same reflector convention
void cpqr_inplace(Workspace& ws, int64_t m, int64_t n, double* W, int64_t ld, int64_t k, int64_t* pivots,
                  double* tau, int* d_flags, long long* d_recomputes, bool padded, cudaStream_t st,
                  bool nopivot = false);
// Panel (delayed-update) CPQR for short-wide padded matrices (cpqr_panel.cu):
// same contract as cpqr_inplace; supported when ld % 64 == 0, ld <= 512 and
// rows [m, ld) are zero.
bool cpqr_panel_supported(int64_t m, int64_t n, int64_t ld, bool padded);
void cpqr_panel(Workspace& ws, int64_t m, int64_t n, double* W, int64_t ld, int64_t k, int64_t* pivots,
                double* tau, int* d_flags, long long* d_recomputes, cudaStream_t st);
// s (k x n, lds) = top k rows of W with strict lower part zeroed and the sign fix
void cpqr_extract_s(int64_t m, int64_t n, const double* W, int64_t ld, int64_t k, double* s, int64_t lds,
                    cudaStream_t st);
// q (m x k) = H_0 .. H_{k-1} [I; 0] with the sign fix of cpqr.hpp:105-112
void cpqr_form_q(int64_t m, int64_t n, const double* W, int64_t ld, int64_t k, const double* tau, double* q,
                 int64_t ldq, cudaStream_t st);

// ---------------------------------------------------------------- triangular / small dense
// Mt (k x k) = transpose of the back-substitution operator of solve.hpp:62-89
// applied to the identity: rows with |d_i| <= thr*max|d| are zero.  s11 may
// carry row sign flips (ignored: they cancel).  zero_rows (k ints) marks them.
void backsub_operator_t(int64_t k, const double* s11, int64_t ld11, double threshold, double* Mt, int* zero_rows,
                        cudaStream_t st);
// diag stats of an upper-triangular block: out[0]=max|d|, out[1]=min|d|
void diag_absminmax(int64_t k, const double* s11, int64_t ld11, double* out, cudaStream_t st);
// strict-lower part nonzero / nonfinite flags for a k x k block (flags[0]: lower nonzero, flags[1]: nonfinite)
void check_upper_triangular(int64_t k, const double* s11, int64_t ld11, int* flags, cudaStream_t st);
// max |x| over an m x n block -> out[0]
void max_abs(int64_t m, int64_t n, const double* a, int64_t lda, double* partials, double* out, cudaStream_t st);
// residual check rows for the singularity test: res[i] = max_c |S12(i,c) - sum_{j>i} S11(i,j) T(j,c)|
void backsub_residual_rows(int64_t k, int64_t nc, const double* s11, int64_t ld11, const double* s12,
                           int64_t ld12, const double* t, int64_t ldt, const int* zero_rows, double* res,
                           cudaStream_t st);
// Cholesky G = R^T R (upper R, k x k, in place on a copy); info[0] = first failing column+1 or 0
void cholesky_upper(Workspace& ws, int64_t k, double* g, int64_t ldg, int* info, cudaStream_t st);
// batched conjugate gradients (solve.hpp:37-57), one column per warp; x, r, d
// k x nc with leading dimension ld, state 3 doubles per column (rho, stop, active)
void cg_init(int64_t k, int64_t nc, int64_t ld, const double* rhs, int64_t ldr, double* x, double* r, double* d, double* state,
             cudaStream_t st);
void cg_step(int64_t k, int64_t nc, int64_t ld, const double* nd, double* x, double* r, double* d, double* state, int* n_active,
             cudaStream_t st);
// inverse of an upper-triangular R (k x k) -> Rinv (upper)
void tri_upper_inverse(int64_t k, const double* r, int64_t ldr, double* rinv, int64_t ldi, cudaStream_t st);
// same for a nonzero diagonal (no singular-row handling), blocked: CholeskyQR factors
void tri_upper_inverse_blocked(int64_t k, const double* r, int64_t ldr, double* rinv, int64_t ldi,
                               cudaStream_t st);

// ---------------------------------------------------------------- Ozaki-II FP64 emulation on INT8 tcgen05
constexpr int kOzakiModuli = 16;
// Scaled residue planes of a K x cols operand (K contiguous): planes[t] is an
// int8 matrix (ld bytes per column) of x' mod m_t, x' = rint(x 2^shift[col]).
struct OzakiOperand {
  int8_t* planes = nullptr;
  int* shift = nullptr;
  int64_t K = 0, cols = 0, ld = 0, plane_stride = 0;
  int beta = 0;
  // residues in [0, m) read as u8 (cheaper split) instead of symmetric s8;
  // allowed on one operand of a product when K <= kOzakiMaxKUnsigned
  bool unsigned_res = false;
};
constexpr int64_t kOzakiMaxKUnsigned = 65536;  // K * 255 * 128 < 2^31
int ozaki_beta(int64_t K);
size_t ozaki_plane_bytes(int64_t K, int64_t cols);
void ozaki_split(int64_t K, int64_t cols, const double* X, int64_t ldx, int beta, OzakiOperand& op, cudaStream_t st);
// split X into an already laid-out operand (op.K, op.cols, op.ld, op.plane_stride, op.beta set)
void ozaki_split_into(const double* X, int64_t ldx, const OzakiOperand& op, cudaStream_t st);
// columns [off, off + cols) of an operand as an operand of its own (same planes)
OzakiOperand ozaki_cols(const OzakiOperand& op, int64_t off, int64_t cols);
// out (M x N) = alpha P^T Q + beta out, reconstructed from 16 INT8 GEMMs
void ozaki_gemm_tn(Workspace& ws, const OzakiOperand& P, const OzakiOperand& Q, int64_t M, int64_t N, double* out,
                   int64_t ldo, double alpha, double beta, cudaStream_t st);

// out (A.K x N) = A_int Q: the contraction over the COLUMNS of the split operand A (its planes are the
// M-major operand); A's column scales folded into Q's rows beforehand (ozaki_fold_scales), Q split
// with ozaki_partner_beta(A.cols, A.beta) bits; zero_shift: A.K zero ints
void ozaki_gemm_a_cols(Workspace& ws, const OzakiOperand& A, const OzakiOperand& Q, int64_t N, double* out,
                       int64_t ldo, const int* zero_shift, cudaStream_t st);
void ozaki_fold_scales(int64_t K, int64_t cols, const double* X, int64_t ldx, const int* shift, double* out,
                       int64_t ldo, cudaStream_t st);
int ozaki_partner_beta(int64_t K, int beta_a);

// ---------------------------------------------------------------- sparse (config 5)
// CSR (m x n, int64 indices) -> CSC with rows ascending within each column
void csr_to_csc(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int64_t* col_idx, const double* val,
                int64_t* col_ptr, int64_t* row_idx, double* cval, cudaStream_t st);
// out (p x n) = B (p x m) A for A in CSC (fixed per-column summation order)
void spmm_csc(int64_t p, int64_t n, const double* B, int64_t ldb, const int64_t* col_ptr, const int64_t* row_idx,
              const double* val, double* out, int64_t ldo, cudaStream_t st);
// compressed segments sel[0..k) (columns of a CSC / rows of a CSR) -> new (k+1) ptr, idx, val
void sparse_select(int64_t k, const int64_t* ptr, const int64_t* idx, const double* val, const int64_t* sel,
                   int64_t* out_ptr, int64_t* out_idx, double* out_val, cudaStream_t st);
void sparse_scatter_cols(int64_t rows, int64_t k, const int64_t* ptr, const int64_t* idx, const double* val,
                         double* dense, int64_t ld, cudaStream_t st);
void sparse_scatter_rows(int64_t k, int64_t cols, const int64_t* ptr, const int64_t* idx, const double* val,
                         double* dense, int64_t ld, cudaStream_t st);
// per-block partial sums of x .* y (m x n blocks)
void dot_sum(int64_t m, int64_t n, const double* x, int64_t ldx, const double* y, int64_t ldy, double* partials,
             int* num_partials, cudaStream_t st);

// ---------------------------------------------------------------- Jacobi SVD (svd.hpp:39-183 semantics)
// thin SVD of a (m x n, m >= n assumed by caller after transposition):
// u (m x n), sigma (n), v (n x n); returns false if not converged in 60 sweeps
bool jacobi_svd(Workspace& ws, int64_t m, int64_t n, const double* a, int64_t lda, double* u, double* sigma,
                double* v, cudaStream_t st);

// bytes (<= a few KB) from device memory to mapped pinned host memory by a
// one-warp kernel (no copy-engine queueing behind bulk transfers)
void copy_bytes_mapped(void* dst, const void* src, size_t bytes, cudaStream_t st);

// out = P^T Q (P: K x M, Q: K x N) summed in ascending k without fused
// multiply-add: the host triple-loop arithmetic of the reference's dense
// SRFT fallback, reproduced bit for bit
void gemm_tn_ordered(int M, int N, int K, const double* P, int64_t ldp, const double* Q, int64_t ldq, double* out,
                     int64_t ldo, cudaStream_t st);

// ---------------------------------------------------------------- multi-GPU (shard.cu)
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void nccl_unique_id(unsigned char out[128]);
void* nccl_comm_init(const unsigned char id[128], int nranks, int rank);
void nccl_comm_destroy(void* comm);

// The collectives of the column-sharded entry points, on the caller's stream.
// Without a communicator (one unsharded rank) they are local no-ops / copies.
struct ShardComm {
  void* comm = nullptr;  // ncclComm_t
  int nranks = 1, rank = 0;
  void all_gather_bytes(const void* send, void* recv, size_t bytes_per_rank, cudaStream_t st) const;
  void all_reduce_sum(double* buf, size_t count, cudaStream_t st) const;
  void all_reduce_sum(int64_t* buf, size_t count, cudaStream_t st) const;
  void all_reduce_max(double* buf, size_t count, cudaStream_t st) const;
};

// cpqr.hpp:32-114 on a column-sharded short-wide matrix (shard.cu header):
// W (m x n_loc, ld) is this rank's block of columns [off, off + n_loc) of an
// m x n_total matrix, overwritten; `steps` steps.  Replicated outputs: perm
// (n_total) and the sign-fixed top `krows` rows of R in logical column order
// S (krows x n_total, ld lds).
void cpqr_sharded(Workspace& ws, const ShardComm& comm, int64_t m, int64_t n_loc, int64_t off, int64_t n_total,
                  double* W, int64_t ld, int64_t steps, int64_t krows, int64_t* perm, double* S, int64_t lds,
                  int* d_flags, long long* d_recomputes, cudaStream_t st);
// the same protocol over `nshards` column blocks of one matrix in one process
// (test vehicle for the multi-rank logic on one GPU; kernels run in sequence)
void cpqr_sharded_emulated(Workspace& ws, int nshards, int64_t m, int64_t n, double* W, int64_t ld, int64_t steps,
                           int64_t krows, int64_t* perm, double* S, int64_t lds, int* d_flags,
                           long long* d_recomputes, cudaStream_t st);

// helpers of the sharded pipeline: owned slot of each global pivot (-1 when
// another rank owns it), inverse permutation, basis() rows of owned columns
void owned_index(const int64_t* perm, int64_t k, int64_t off, int64_t n_loc, int64_t* idx, cudaStream_t st);
void inverse_perm(const int64_t* perm, int64_t n, int64_t* inv, cudaStream_t st);
void basis_rows(const int64_t* inv, int64_t off, int64_t n_loc, int64_t k, const double* coeff, int64_t ldc,
                double* B, cudaStream_t st);

// verify.cu: out(piv[l], :) = l < k ? (top ? top(l, :) : 0) : res(l - k, :) for an m x b block
void scatter_stack(int64_t m, int64_t b, int64_t k, const int64_t* piv, const double* top, int64_t ldt,
                   const double* res, int64_t ldr, double* out, int64_t ldo, cudaStream_t st);

}  // namespace lrb
