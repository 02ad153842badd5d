// small.cu -- k x k triangular and small dense kernels that sit between the
// big contractions: the back-substitution operator of solve.hpp:62-89,
// escalation statistics (solve.hpp:119-126), the singularity residual test
// (solve.hpp:75-83), Cholesky for CholeskyQR2 and triangular inverses.
// These are latency-bound (k <= a few thousand); each uses one warp per
// column with a fixed reduction order so results are reproducible.
#include "common.cuh"
#include "kernels.h"

namespace lrb {

namespace {

__device__ double block_max_abs_diag(int64_t k, const double* s11, int64_t ld11, double* sh) {
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) mx = fmax(mx, fabs(s11[i + i * ld11]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, sh[w]);
  __syncthreads();
  return t;
}

// One warp per column c of the operator M = backsub(S11, I) (col-major k x k):
//   for i = c..0: rhs = delta(i,c) - sum_{j>i} S11(i,j) M(j,c)  (j ascending)
//                 M(i,c) = |d_i| <= tol ? 0 : rhs / d_i
__global__ void backsub_operator_kernel(int64_t k, const double* __restrict__ s11, int64_t ld11, double threshold,
                                        double* __restrict__ M, int* __restrict__ zero_rows) {
  __shared__ double sh[32];
  const double tol = threshold * block_max_abs_diag(k, s11, ld11, sh);
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
  if (blockIdx.x == 0)
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) zero_rows[i] = fabs(s11[i + i * ld11]) <= tol;
  if (c >= k) return;
  double* mc = M + c * k;
  for (int64_t i = c + 1 + lane; i < k; i += 32) mc[i] = 0.0;
  for (int64_t i = c; i >= 0; --i) {
    double acc = 0.0;
    for (int64_t j = i + 1 + lane; j <= c; j += 32) acc = fma(s11[i + j * ld11], mc[j], acc);
    acc = warp_sum(acc);
    if (lane == 0) {
      const double d = s11[i + i * ld11];
      const double rhs = (i == c ? 1.0 : 0.0) - acc;
      mc[i] = fabs(d) <= tol ? 0.0 : rhs / d;
    }
    __syncwarp();
  }
}

// Same operator, column-oriented ("axpy") form with the right-hand side held in
// shared memory: for i = c..0: M(i,c) = x_i / d_i (or 0 for a zeroed row), then
// x_j -= S11(j,i) M(i,c) for j < i.  S11's column i is contiguous, so each
// step is one coalesced read (prefetched a step ahead) instead of a strided
// row walk.  One warp per column; x for up to kAxpyMaxK rows.
constexpr int kAxpyMaxK = 2048;
constexpr int kAxpyWarps = 4;

__global__ void backsub_operator_axpy_kernel(int64_t k, const double* __restrict__ s11, int64_t ld11,
                                             double threshold, double* __restrict__ M, int* __restrict__ zero_rows) {
  extern __shared__ double xs_all[];
  __shared__ double sh[32];
  const double tol = threshold * block_max_abs_diag(k, s11, ld11, sh);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * kAxpyWarps + w;
  if (blockIdx.x == 0)
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) zero_rows[i] = fabs(s11[i + i * ld11]) <= tol;
  if (c >= k) return;
  double* x = xs_all + (int64_t)w * k;
  for (int64_t i = lane; i <= c; i += 32) x[i] = (i == c) ? 1.0 : 0.0;
  double* mc = M + c * k;
  for (int64_t i = c + 1 + lane; i < k; i += 32) mc[i] = 0.0;
  __syncwarp();
  // prefetch column c of S11 (rows < c) in 32-row chunks held per lane
  for (int64_t i = c; i >= 0; --i) {
    const double d = s11[i + i * ld11];
    const double mi = fabs(d) <= tol ? 0.0 : x[i] / d;
    if (lane == 0) mc[i] = mi;
    if (mi != 0.0) {
      const double* col = s11 + i * ld11;
      for (int64_t j = lane; j < i; j += 32) x[j] = fma(-col[j], mi, x[j]);
    }
    __syncwarp();
  }
}

// Register-pipelined variant for k <= 512: column i-1 of S11 (rows < i-1) and
// its diagonal are loaded while the axpy of column i runs, so each step costs
// a few shared-memory ops instead of an L2 round trip.  Same arithmetic order.
constexpr int kPipeMaxK = 512;
__global__ void backsub_operator_pipe_kernel(int64_t k, const double* __restrict__ s11, int64_t ld11,
                                             double threshold, double* __restrict__ M, int* __restrict__ zero_rows) {
  extern __shared__ double xs_all[];
  __shared__ double sh[32];
  const double tol = threshold * block_max_abs_diag(k, s11, ld11, sh);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * kAxpyWarps + w;
  if (blockIdx.x == 0)
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) zero_rows[i] = fabs(s11[i + i * ld11]) <= tol;
  if (c >= k) return;
  double* x = xs_all + (int64_t)w * k;
  for (int64_t i = lane; i <= c; i += 32) x[i] = (i == c) ? 1.0 : 0.0;
  double* mc = M + c * k;
  for (int64_t i = c + 1 + lane; i < k; i += 32) mc[i] = 0.0;
  constexpr int T = kPipeMaxK / 32;
  double cur[T], nxt[T];
  auto load = [&](int64_t i, double (&v)[T]) {
    const double* col = s11 + i * ld11;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int64_t j = lane + 32 * t;
      v[t] = j < i ? col[j] : 0.0;
    }
  };
  load(c, cur);
  double d = s11[c + c * ld11];
  __syncwarp();
  for (int64_t i = c; i >= 0; --i) {
    double dn = 0.0;
    if (i > 0) {
      load(i - 1, nxt);
      dn = s11[(i - 1) + (i - 1) * ld11];
    }
    const double mi = fabs(d) <= tol ? 0.0 : x[i] / d;
    if (lane == 0) mc[i] = mi;
    if (mi != 0.0) {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int64_t j = lane + 32 * t;
        if (j < i) x[j] = fma(-cur[t], mi, x[j]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < T; ++t) cur[t] = nxt[t];
    d = dn;
  }
}

__global__ void diag_minmax_kernel(int64_t k, const double* __restrict__ s11, int64_t ld11, double* out) {
  __shared__ double smx[32], smn[32];
  double mx = 0.0, mn = INFINITY;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
    const double d = fabs(s11[i + i * ld11]);
    mx = fmax(mx, d);
    mn = fmin(mn, d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if ((threadIdx.x & 31) == 0) { smx[threadIdx.x >> 5] = mx; smn[threadIdx.x >> 5] = mn; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a = fmax(a, smx[w]); b = fmin(b, smn[w]); }
    out[0] = a;
    out[1] = b;
  }
}

__global__ void check_upper_kernel(int64_t k, const double* __restrict__ s11, int64_t ld11, int* flags) {
  int lower = 0, bad = 0;
  const int64_t total = k * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % k, j = t / k;
    const double x = s11[i + j * ld11];
    bad |= !isfinite(x);
    lower |= (i > j) && (x != 0.0);
  }
  if (__syncthreads_or(lower) && threadIdx.x == 0) atomicOr(flags + 0, 1);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags + 1, 1);
}

// res[i] (only for zero rows) = max_c |S12(i,c) - sum_{j>i} S11(i,j) T(j,c)|, as per-block partial maxima
__global__ void backsub_residual_kernel(int64_t k, int64_t nc, const double* __restrict__ s11, int64_t ld11,
                                        const double* __restrict__ s12, int64_t ld12, const double* __restrict__ t,
                                        int64_t ldt, int64_t row, double* __restrict__ partial) {
  double mx = 0.0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    double rhs = s12[row + c * ld12];
    for (int64_t j = row + 1; j < k; ++j) rhs -= s11[row + j * ld11] * t[j + c * ldt];
    mx = fmax(mx, fabs(rhs));
  }
  __shared__ double sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a = fmax(a, sh[w]);
    partial[blockIdx.x] = a;
  }
}

__global__ void max_reduce_kernel(const double* __restrict__ p, int n, double* out) {
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < n; ++i) a = fmax(a, p[i]);
    out[0] = a;
  }
}

// ---- blocked Cholesky (G = R^T R, upper): diagonal block in shared memory,
// panel by forward substitution, trailing SYRK on the DMMA GEMM.
constexpr int kCholB = 64;

__global__ void chol_diag_kernel(int64_t j0, int jb, double* __restrict__ g, int64_t ldg, int* info) {
  // 256 threads own fixed 4x4 element sets (rows tr + 16u, columns tc + 16v)
  // in registers; per column j the owners of row j scale it and publish it in
  // shared memory (with one rsqrt per thread), then every thread applies the
  // rank-1 update to its registers and the owner of the next diagonal entry
  // publishes it.  Same arithmetic as scaling the row first.
  __shared__ double srow[kCholB];
  __shared__ double sd;
  __shared__ int fail;
  if (info[0] != 0) return;
  const int tr = threadIdx.x & 15, tc = threadIdx.x >> 4;
  double reg[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = tr + 16 * u, c = tc + 16 * v;
      reg[u][v] = (r <= c && c < jb) ? g[(j0 + r) + (j0 + c) * ldg] : 0.0;
    }
  if (threadIdx.x == 0) {
    fail = 0;
    sd = g[j0 + j0 * ldg];
  }
  __syncthreads();
  bool stop = false;
#pragma unroll
  for (int U = 0; U < 4; ++U) {
    for (int jj = 0; jj < 16 && !stop; ++jj) {
      const int j = 16 * U + jj;
      if (j >= jb) {
        stop = true;
        break;
      }
      const double d = sd;
      if (!(d > 0.0) || !isfinite(d)) {  // uniform
        if (threadIdx.x == 0) fail = j + 1;
        stop = true;
        break;
      }
      const double ri = rsqrt(d);
      if (tr == jj) {  // row j = tr + 16 U
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c = tc + 16 * v;
          if (c > j && c < jb) {
            reg[U][v] *= ri;
            srow[c] = reg[U][v];
          } else if (c == j) {
            reg[U][v] = sqrt(d);
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = tr + 16 * u;
        if (r <= j) continue;
        const double sr = srow[r];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c = tc + 16 * v;
          if (r <= c && c < jb) reg[u][v] = fma(-sr, srow[c], reg[u][v]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (tr == tc && tr + 16 * u == j + 1) sd = reg[u][u];
      __syncthreads();
    }
  }
  if (fail) {
    if (threadIdx.x == 0) info[0] = (int)(j0 + fail);
    return;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = tr + 16 * u, c = tc + 16 * v;
      if (r < jb && c < jb) g[(j0 + r) + (j0 + c) * ldg] = r <= c ? reg[u][v] : 0.0;
    }
}

// C = beta C + alpha A^T B (column-major, small K): the Cholesky trailing update
__global__ void gemm_tn_small_kernel(int m, int n, int kk, double alpha, const double* __restrict__ A, int64_t lda,
                                     const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C,
                                     int64_t ldc, bool upper_only) {
  __shared__ double As[32][33];  // As[l][i] = A(l0 + l, i0 + i)
  __shared__ double Bs[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  if (upper_only && i0 > j0 + 31) return;
  const int ti = threadIdx.x & 31, tj = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int l0 = 0; l0 < kk; l0 += 32) {
    for (int t = threadIdx.x; t < 32 * 32; t += blockDim.x) {
      const int a = t & 31, b = t >> 5;
      As[a][b] = (l0 + a < kk && i0 + b < m) ? A[(l0 + a) + (int64_t)(i0 + b) * lda] : 0.0;
      Bs[a][b] = (l0 + a < kk && j0 + b < n) ? B[(l0 + a) + (int64_t)(j0 + b) * ldb] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int l = 0; l < 32; ++l) {
      const double av = As[l][ti];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(av, Bs[l][tj + 8 * q], acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + ti, j = j0 + tj + 8 * q;
    if (i < m && j < n && (!upper_only || i <= j)) {
      double* cp = C + i + (int64_t)j * ldc;
      *cp = beta == 0.0 ? alpha * acc[q] : fma(alpha, acc[q], beta * *cp);
    }
  }
}

// Panel by forward substitution, one warp per column (axpy form, two rows per
// lane in registers): X(i) = G(i) / R(i,i), then G(l) -= R(i,l) X(i) for l > i.
__global__ void chol_panel_warp_kernel(int64_t k, int64_t j0, int jb, double* __restrict__ g, int64_t ldg,
                                       const int* info) {
  __shared__ double r[kCholB][kCholB + 1];
  if (info[0] != 0) return;
  for (int t = threadIdx.x; t < jb * jb; t += blockDim.x) {
    const int i = t % jb, j = t / jb;
    r[i][j] = g[(j0 + i) + (j0 + j) * ldg];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t c = j0 + jb + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= k) return;
  double* col = g + c * ldg + j0;
  double x0 = lane < jb ? col[lane] : 0.0;
  double x1 = lane + 32 < jb ? col[lane + 32] : 0.0;
  for (int i = 0; i < jb; ++i) {
    const double raw = __shfl_sync(0xffffffffu, i < 32 ? x0 : x1, i & 31);
    const double xi = raw / r[i][i];
    if (lane == (i & 31)) {
      if (i < 32) x0 = xi;
      else x1 = xi;
    }
    if (lane > i && lane < jb) x0 = fma(-r[i][lane], xi, x0);
    if (lane + 32 > i && lane + 32 < jb) x1 = fma(-r[i][lane + 32], xi, x1);
  }
  if (lane < jb) col[lane] = x0;
  if (lane + 32 < jb) col[lane + 32] = x1;
}

__global__ void zero_strict_lower_kernel(int64_t k, double* __restrict__ g, int64_t ldg) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < k * k; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % k, j = t / k;
    if (i > j) g[i + j * ldg] = 0.0;
  }
}

// Right-looking Cholesky G = R^T R on the upper triangle, one CTA (small k).
__global__ void cholesky_upper_kernel(int64_t k, double* __restrict__ g, int64_t ldg, int* info) {
  __shared__ double sdiag;
  __shared__ int sfail;
  if (threadIdx.x == 0) sfail = 0;
  __syncthreads();
  for (int64_t j = 0; j < k; ++j) {
    if (threadIdx.x == 0) {
      const double d = g[j + j * ldg];
      if (!(d > 0.0) || !isfinite(d)) {
        sfail = 1;
        info[0] = (int)(j + 1);
      } else {
        sdiag = sqrt(d);
        g[j + j * ldg] = sdiag;
      }
    }
    __syncthreads();
    if (sfail) return;
    const double rd = sdiag;
    for (int64_t c = j + 1 + threadIdx.x; c < k; c += blockDim.x) g[j + c * ldg] /= rd;
    __syncthreads();
    // trailing update of the upper triangle: G(a,b) -= R(j,a) R(j,b), j < a <= b
    const int64_t nt = k - j - 1;
    const int64_t tot = nt * nt;
    for (int64_t t = threadIdx.x; t < tot; t += blockDim.x) {
      const int64_t a = j + 1 + t % nt, b = j + 1 + t / nt;
      if (a <= b) g[a + b * ldg] = fma(-g[j + a * ldg], g[j + b * ldg], g[a + b * ldg]);
    }
    __syncthreads();
  }
  // zero the strict lower part so R is a clean upper-triangular factor
  for (int64_t t = threadIdx.x; t < k * k; t += blockDim.x) {
    const int64_t a = t % k, b = t / k;
    if (a > b) g[a + b * ldg] = 0.0;
  }
  if (threadIdx.x == 0) info[0] = 0;
}

void launch_backsub_operator(int64_t k, const double* s11, int64_t ld11, double threshold, double* M, int* zr,
                             cudaStream_t st) {
  if (k <= kPipeMaxK) {
    const size_t smem = sizeof(double) * kAxpyWarps * (size_t)k;
    backsub_operator_pipe_kernel<<<(unsigned)((k + kAxpyWarps - 1) / kAxpyWarps), kAxpyWarps * 32, smem, st>>>(
        k, s11, ld11, threshold, M, zr);
  } else if (k <= kAxpyMaxK) {
    const size_t smem = sizeof(double) * kAxpyWarps * (size_t)k;
    static bool attr = false;
    if (!attr) {
      LRB_CUDA(cudaFuncSetAttribute(backsub_operator_axpy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(sizeof(double) * kAxpyWarps * kAxpyMaxK)));
      attr = true;
    }
    backsub_operator_axpy_kernel<<<(unsigned)((k + kAxpyWarps - 1) / kAxpyWarps), kAxpyWarps * 32, smem, st>>>(
        k, s11, ld11, threshold, M, zr);
  } else {
    const int wpb = 8;
    backsub_operator_kernel<<<(unsigned)((k + wpb - 1) / wpb), wpb * 32, 0, st>>>(k, s11, ld11, threshold, M, zr);
  }
  LRB_CHECK_LAUNCH();
}

}  // namespace

void backsub_operator_t(int64_t k, const double* s11, int64_t ld11, double threshold, double* Mt, int* zero_rows,
                        cudaStream_t st) {
  // M is written col-major into Mt's storage first, then transposed in place via a temp
  double* tmp = nullptr;
  LRB_CUDA(cudaMallocAsync(&tmp, sizeof(double) * k * k, st));
  launch_backsub_operator(k, s11, ld11, threshold, tmp, zero_rows, st);
  transpose_matrix(k, k, tmp, k, Mt, k, st);
  LRB_CUDA(cudaFreeAsync(tmp, st));
}

void diag_absminmax(int64_t k, const double* s11, int64_t ld11, double* out, cudaStream_t st) {
  diag_minmax_kernel<<<1, 256, 0, st>>>(k, s11, ld11, out);
  LRB_CHECK_LAUNCH();
}

void check_upper_triangular(int64_t k, const double* s11, int64_t ld11, int* flags, cudaStream_t st) {
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((k * k + 255) / 256, 4 * num_sms()));
  check_upper_kernel<<<g, 256, 0, st>>>(k, s11, ld11, flags);
  LRB_CHECK_LAUNCH();
}

void backsub_residual_rows(int64_t k, int64_t nc, const double* s11, int64_t ld11, const double* s12, int64_t ld12,
                           const double* t, int64_t ldt, const int* zero_rows_host, double* res, cudaStream_t st) {
  // zero_rows_host: host array; res: device array of k (only zero rows written)
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((nc + 255) / 256, 2 * num_sms()));
  double* partial = nullptr;
  LRB_CUDA(cudaMallocAsync(&partial, sizeof(double) * g, st));
  for (int64_t i = k - 1; i >= 0; --i) {
    if (!zero_rows_host[i]) continue;
    backsub_residual_kernel<<<g, 256, 0, st>>>(k, nc, s11, ld11, s12, ld12, t, ldt, i, partial);
    LRB_CHECK_LAUNCH();
    max_reduce_kernel<<<1, 32, 0, st>>>(partial, g, res + i);
    LRB_CHECK_LAUNCH();
  }
  LRB_CUDA(cudaFreeAsync(partial, st));
}

// ---------------------------------------------------------------- batched CG
// solve.hpp:37-57 (detail::conjugate_gradient) for every column j of the
// right-hand side at once: one warp per column keeps its x, r, d (k entries,
// ld k) and (rho, stop, active); the k x k products normal * D of all
// columns are one GEMM between iterations.  Column semantics as the
// reference: x = 0, r = d = rhs, stop = 1e-28 ||rhs||^2, iterate while
// it < max_iters and rho > stop, leave on denom = d.(normal d) <= 0.
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void cg_init_kernel(int64_t k, int64_t nc, int64_t ld, const double* __restrict__ rhs, int64_t ldr,
                               double* __restrict__ x, double* __restrict__ r, double* __restrict__ d,
                               double* __restrict__ st) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= nc) return;
  double acc = 0.0;
  for (int64_t i = lane; i < k; i += 32) {
    const double b = rhs[j * ldr + i];
    x[j * ld + i] = 0.0;
    r[j * ld + i] = b;
    d[j * ld + i] = b;
    acc += b * b;
  }
  acc = warp_sum_d(acc);
  if (lane == 0) {
    st[3 * j] = acc;              // rho
    st[3 * j + 1] = 1e-28 * acc;  // stop
    st[3 * j + 2] = acc > 1e-28 * acc ? 1.0 : 0.0;
  }
}

__global__ void cg_step_kernel(int64_t k, int64_t nc, int64_t ld, const double* __restrict__ nd, double* __restrict__ x,
                               double* __restrict__ r, double* __restrict__ d, double* __restrict__ st,
                               int* __restrict__ n_active) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= nc || st[3 * j + 2] == 0.0) return;
  double den = 0.0;
  for (int64_t i = lane; i < k; i += 32) den += d[j * ld + i] * nd[j * ld + i];
  den = warp_sum_d(den);
  if (den <= 0.0) {
    if (lane == 0) st[3 * j + 2] = 0.0;
    return;
  }
  const double rho = st[3 * j], alpha = rho / den;
  double rn = 0.0;
  for (int64_t i = lane; i < k; i += 32) {
    x[j * ld + i] += alpha * d[j * ld + i];
    const double ri = r[j * ld + i] - alpha * nd[j * ld + i];
    r[j * ld + i] = ri;
    rn += ri * ri;
  }
  rn = warp_sum_d(rn);
  const double beta = rn / rho;
  for (int64_t i = lane; i < k; i += 32) d[j * ld + i] = r[j * ld + i] + beta * d[j * ld + i];
  if (lane == 0) {
    st[3 * j] = rn;
    const bool act = rn > st[3 * j + 1];
    st[3 * j + 2] = act ? 1.0 : 0.0;
    if (act) atomicAdd(n_active, 1);
  }
}

void cg_init(int64_t k, int64_t nc, int64_t ld, const double* rhs, int64_t ldr, double* x, double* r, double* d, double* state,
             cudaStream_t st) {
  const int64_t g = (nc * 32 + 255) / 256;
  cg_init_kernel<<<(unsigned)g, 256, 0, st>>>(k, nc, ld, rhs, ldr, x, r, d, state);
  LRB_CHECK_LAUNCH();
}

void cg_step(int64_t k, int64_t nc, int64_t ld, const double* nd, double* x, double* r, double* d, double* state, int* n_active,
             cudaStream_t st) {
  const int64_t g = (nc * 32 + 255) / 256;
  cg_step_kernel<<<(unsigned)g, 256, 0, st>>>(k, nc, ld, nd, x, r, d, state, n_active);
  LRB_CHECK_LAUNCH();
}

void cholesky_upper(Workspace& ws, int64_t k, double* g, int64_t ldg, int* info, cudaStream_t st) {
  if (k <= 2 * kCholB || (ldg & 1) || (reinterpret_cast<uintptr_t>(g) & 15)) {
    cholesky_upper_kernel<<<1, 1024, 0, st>>>(k, g, ldg, info);
    LRB_CHECK_LAUNCH();
    return;
  }
  LRB_CUDA(cudaMemsetAsync(info, 0, sizeof(int), st));
  for (int64_t j0 = 0; j0 < k; j0 += kCholB) {
    const int jb = (int)std::min<int64_t>(kCholB, k - j0);
    chol_diag_kernel<<<1, 256, 0, st>>>(j0, jb, g, ldg, info);
    LRB_CHECK_LAUNCH();
    const int64_t nt = k - j0 - jb;
    if (nt <= 0) break;
    chol_panel_warp_kernel<<<(unsigned)((nt + 7) / 8), 256, 0, st>>>(k, j0, jb, g, ldg, info);
    LRB_CHECK_LAUNCH();
    // G(J+, J+) -= X^T X with X = R(J, J+) (jb x nt): TN GEMM with K = jb
    const double* X = g + j0 + (j0 + jb) * ldg;
    double* T = g + (j0 + jb) + (j0 + jb) * ldg;
    (void)ws;
    gemm_tn_small_kernel<<<dim3((unsigned)((nt + 31) / 32), (unsigned)((nt + 31) / 32)), 256, 0, st>>>(
        (int)nt, (int)nt, jb, -1.0, X, ldg, X, ldg, 1.0, T, ldg, true);
    LRB_CHECK_LAUNCH();
  }
  zero_strict_lower_kernel<<<(unsigned)std::min<int64_t>((k * k + 255) / 256, 4096), 256, 0, st>>>(k, g, ldg);
  LRB_CHECK_LAUNCH();
}

namespace {
constexpr int kInvB = 64;

// inverse of each kInvB diagonal block: thread c back-substitutes column c
__global__ void tri_inv_leaf_kernel(int64_t k, const double* __restrict__ r, int64_t ldr, double* __restrict__ ri,
                                    int64_t ldi) {
  extern __shared__ double inv_smem[];
  auto a = reinterpret_cast<double(*)[kInvB + 1]>(inv_smem);
  auto x = reinterpret_cast<double(*)[kInvB + 1]>(inv_smem + kInvB * (kInvB + 1));
  const int64_t b0 = (int64_t)blockIdx.x * kInvB;
  const int nb = (int)(k - b0 < kInvB ? k - b0 : kInvB);
  for (int t = threadIdx.x; t < kInvB * kInvB; t += blockDim.x) {
    const int i = t % kInvB, j = t / kInvB;
    a[i][j] = (i < nb && j < nb) ? r[(b0 + i) + (b0 + j) * ldr] : 0.0;
  }
  __syncthreads();
  const int c = threadIdx.x;
  if (c < nb) {
    for (int i = c; i >= 0; --i) {
      double v = i == c ? 1.0 : 0.0;
      for (int l = i + 1; l <= c; ++l) v = fma(-a[i][l], x[l][c], v);
      x[i][c] = v / a[i][i];
    }
    for (int i = 0; i < nb; ++i) ri[(b0 + i) + (b0 + c) * ldi] = i <= c ? x[i][c] : 0.0;
  }
}

// One level of the blocked triangular inverse for every diagonal pair at once
// (blockIdx.z = pair at p0 = 2 h z; sizes h x hc, hc = min(h, k - p0 - h)):
// step 0: T_z = R(p0:p0+h, p0+h:p0+h+hc) Rinv(p0+h.., p0+h..)   (h x hc, K = hc)
// step 1: Rinv(p0:p0+h, p0+h..) = -Rinv(p0.., p0..) T_z          (h x hc, K = h)
// 32x32 output tiles, 256 threads x 4 outputs, K in 32-deep shared-memory slices.
__global__ void tri_inv_level_kernel(int step, int64_t h, int64_t k, const double* __restrict__ r, int64_t ldr,
                                     double* __restrict__ ri, int64_t ldi, double* __restrict__ T) {
  __shared__ double As[32][33];
  __shared__ double Bs[32][33];
  const int64_t p0 = 2 * h * blockIdx.z;
  const int64_t hc = min(h, k - p0 - h);
  if (hc <= 0) return;
  const int m = (int)h, n = (int)hc, kk = step == 0 ? (int)hc : (int)h;
  const double* A = step == 0 ? r + p0 + (p0 + h) * ldr : ri + p0 + p0 * ldi;
  const int64_t lda = step == 0 ? ldr : ldi;
  double* Tz = T + (size_t)blockIdx.z * (size_t)(h * h);
  const double* B = step == 0 ? ri + (p0 + h) + (p0 + h) * ldi : Tz;
  const int64_t ldb = step == 0 ? ldi : h;
  double* C = step == 0 ? Tz : ri + p0 + (p0 + h) * ldi;
  const int64_t ldc = step == 0 ? h : ldi;
  const double alpha = step == 0 ? 1.0 : -1.0;
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  if (i0 >= m || j0 >= n) return;
  const int ti = threadIdx.x & 31, tj = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int l0 = 0; l0 < kk; l0 += 32) {
    for (int t = threadIdx.x; t < 32 * 32; t += blockDim.x) {
      const int a = t & 31, b = t >> 5;
      As[a][b] = (i0 + a < m && l0 + b < kk) ? A[(i0 + a) + (int64_t)(l0 + b) * lda] : 0.0;
      Bs[a][b] = (l0 + a < kk && j0 + b < n) ? B[(l0 + a) + (int64_t)(j0 + b) * ldb] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int l = 0; l < 32; ++l) {
      const double av = As[ti][l];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(av, Bs[l][tj + 8 * q], acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + ti, j = j0 + tj + 8 * q;
    if (i < m && j < n) C[i + (int64_t)j * ldc] = alpha * acc[q];
  }
}
}  // namespace

namespace {
// out = P^T Q with every entry summed in ascending k as fl(acc + fl(p q)) --
// no fused multiply-add, the arithmetic of a plain host triple loop (the
// reference's dense SRFT fallback is such a product, sketch.hpp:137-141)
__global__ void gemm_tn_ordered_kernel(int M, int N, int K, const double* __restrict__ P, int64_t ldp,
                                       const double* __restrict__ Q, int64_t ldq, double* __restrict__ out,
                                       int64_t ldo) {
  __shared__ double Ps[32][33];  // Ps[k][i] = P(k0 + k, i0 + i)
  __shared__ double Qs[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const int ti = threadIdx.x & 31, tj = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int t = threadIdx.x; t < 32 * 32; t += blockDim.x) {
      const int kk = t & 31, b = t >> 5;
      Ps[kk][b] = (k0 + kk < K && i0 + b < M) ? P[(k0 + kk) + (int64_t)(i0 + b) * ldp] : 0.0;
      Qs[kk][b] = (k0 + kk < K && j0 + b < N) ? Q[(k0 + kk) + (int64_t)(j0 + b) * ldq] : 0.0;
    }
    __syncthreads();
    const int kn = K - k0 < 32 ? K - k0 : 32;
    for (int kk = 0; kk < kn; ++kk) {
      const double pv = Ps[kk][ti];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(pv, Qs[kk][tj + 8 * q]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + ti, j = j0 + tj + 8 * q;
    if (i < M && j < N) out[i + (int64_t)j * ldo] = acc[q];
  }
}
}  // namespace

void gemm_tn_ordered(int M, int N, int K, const double* P, int64_t ldp, const double* Q, int64_t ldq, double* out,
                     int64_t ldo, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  gemm_tn_ordered_kernel<<<dim3((M + 31) / 32, (N + 31) / 32), 256, 0, st>>>(M, N, K, P, ldp, Q, ldq, out, ldo);
  LRB_CHECK_LAUNCH();
}

// R^-1 of an upper-triangular R with a nonzero diagonal by blocks: diagonal
// blocks by back substitution, then [A B; 0 C]^-1 = [A^-1, -A^-1 B C^-1; 0, C^-1]
// level by level (the serial chain is kInvB steps, not k).
void tri_upper_inverse_blocked(int64_t k, const double* r, int64_t ldr, double* rinv, int64_t ldi,
                               cudaStream_t st) {
  LRB_CUDA(cudaMemset2DAsync(rinv, sizeof(double) * ldi, 0, sizeof(double) * k, k, st));
  constexpr int smem = 2 * kInvB * (kInvB + 1) * (int)sizeof(double);
  static bool attr = false;
  if (!attr) {
    LRB_CUDA(cudaFuncSetAttribute(tri_inv_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  tri_inv_leaf_kernel<<<(unsigned)((k + kInvB - 1) / kInvB), kInvB, smem, st>>>(k, r, ldr, rinv, ldi);
  LRB_CHECK_LAUNCH();
  if (k <= kInvB) return;
  double* T = nullptr;
  LRB_CUDA(cudaMallocAsync(&T, sizeof(double) * k * k, st));
  for (int64_t h = kInvB; h < k; h *= 2) {
    // every pair [A B; 0 C] of this level: T = B C^-1, then the block = -A^-1 T
    const unsigned pairs = (unsigned)((k - h + 2 * h - 1) / (2 * h));
    const dim3 grid((unsigned)((h + 31) / 32), (unsigned)((h + 31) / 32), pairs);
    for (int step = 0; step < 2; ++step) {
      tri_inv_level_kernel<<<grid, 256, 0, st>>>(step, h, k, r, ldr, rinv, ldi, T);
      LRB_CHECK_LAUNCH();
    }
  }
  LRB_CUDA(cudaFreeAsync(T, st));
}

void tri_upper_inverse(int64_t k, const double* r, int64_t ldr, double* rinv, int64_t ldi, cudaStream_t st) {
  int* zr = nullptr;
  LRB_CUDA(cudaMallocAsync(&zr, sizeof(int) * k, st));
  double* tmp = nullptr;
  LRB_CUDA(cudaMallocAsync(&tmp, sizeof(double) * k * k, st));
  // threshold 0: only exactly-zero diagonals are treated as singular (rows zeroed)
  launch_backsub_operator(k, r, ldr, 0.0, tmp, zr, st);
  copy_matrix(k, k, tmp, k, rinv, ldi, st);
  LRB_CUDA(cudaFreeAsync(tmp, st));
  LRB_CUDA(cudaFreeAsync(zr, st));
}

}  // namespace lrb
