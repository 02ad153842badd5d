/*
 * lowrank_oracle.c -- CPU restatement of the reference ID / CUR hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see lowrank_oracle.h).  Never linked by the
 * product library.  Each function cites the reference lines it restates
 * (paths relative to /root/reference/proj/include/lowrank unless noted).
 *
 * Eigen (the reference's only dependency, >= 3.4, absent from this image)
 * supplies the GEMV / GEMM / norm arithmetic the reference calls; those are
 * restated here as plain loops with a fixed summation order.  Results
 * therefore agree with an Eigen build to rounding, not bitwise; the pivot
 * sequences agree exactly on the well-separated synthetic spectra.
 */
#include "lowrank_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static _Thread_local char g_err[512];
static _Thread_local int64_t g_sing_index = -1;

const char* lro_last_error(void) { return g_err; }
int64_t lro_last_singular_index(void) { return g_sing_index; }

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

void lro_set_threads(int n) {
#ifdef _OPENMP
  if (n <= 0) n = omp_get_num_procs();
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}

#define IDX(i, j, ld) ((size_t)(i) + (size_t)(j) * (size_t)(ld))
#define NEW(T, n) ((T*)malloc(sizeof(T) * (size_t)((n) > 0 ? (n) : 1)))

/* ---------------------------------------------------------------- rng.hpp */

/* rng.hpp:14-18 */
uint64_t lro_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* rng.hpp:27-29: counter-mode SplitMix64 */
uint64_t lro_stream_value(uint64_t seed, uint64_t index) {
  return lro_mix64(seed + (index + 1) * 0x9E3779B97F4A7C15ULL);
}

/* rng.hpp:32-34 */
uint64_t lro_derive_seed(uint64_t seed, uint64_t tag) {
  return lro_stream_value(seed, tag ^ 0xD1B54A32D192ED03ULL);
}

/* rng.hpp:74-94: Box-Muller over stream pairs in row-major stream order,
 * stored column-major. */
int lro_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  if (rows < 1 || cols < 1)
    return fail(LRO_EINVAL, "gaussian_matrix: dimensions must be positive");
  const int64_t total = rows * cols;
  const double two_pi = 2.0 * 3.14159265358979323846;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < total; i += 2) {
    const uint64_t pair = (uint64_t)i;
    const double u1 = (double)((lro_stream_value(seed, pair) >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(lro_stream_value(seed, pair + 1) >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = two_pi * u2;
    out[IDX(i / cols, i % cols, rows)] = radius * cos(angle);
    if (i + 1 < total) out[IDX((i + 1) / cols, (i + 1) % cols, rows)] = radius * sin(angle);
  }
  return LRO_OK;
}

/* --------------------------------------------------------------- helpers */

static int all_finite(int64_t m, int64_t n, const double* a, int64_t lda) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i)
      if (!isfinite(a[IDX(i, j, lda)])) return 0;
  return 1;
}

/* core.hpp:44-48 */
static int require_nonempty(int64_t m, int64_t n, const char* who) {
  if (m < 1 || n < 1) return fail(LRO_EINVAL, "%s: matrix must be nonempty", who);
  return LRO_OK;
}
/* core.hpp:50-54 */
static int require_finite(int64_t m, int64_t n, const double* a, int64_t lda, const char* who) {
  if (!all_finite(m, n, a, lda)) return fail(LRO_EINVAL, "%s: matrix has non-finite entries", who);
  return LRO_OK;
}
/* core.hpp:56-61 */
static int require_rank_in_range(int64_t k, int64_t rows, int64_t cols, const char* who) {
  const int64_t mn = rows < cols ? rows : cols;
  if (k < 1 || k > mn)
    return fail(LRO_EINVAL, "%s: rank %lld out of range for %lldx%lld matrix", who, (long long)k,
                (long long)rows, (long long)cols);
  return LRO_OK;
}

/* C(i0.., j0..) += A(:, k0..k0+kc) B(k0..k0+kc, j0..) on an mc x nc block.
 * Every output element is updated as c = c + a_k b_k for k ascending, one
 * rounded product and one rounded sum per term (no FMA contraction: the
 * file is built with -ffp-contract=off), so the result is bitwise the plain
 * triple loop's.  Four columns x four k are kept per pass so each c value is
 * loaded and stored once per four terms and each a value feeds four
 * columns; the i loop vectorises (elementwise, no reordering). */
#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
__attribute__((target_clones("avx512f", "avx2", "default")))
#endif
static void gemm_block(int64_t mc, int64_t nc, int64_t kc, const double* restrict A, int64_t lda,
                       const double* restrict B, int64_t ldb, double* restrict C, int64_t ldc) {
  int64_t j = 0;
  for (; j + 4 <= nc; j += 4) {
    double* restrict c0 = C + (size_t)j * ldc;
    double* restrict c1 = c0 + ldc;
    double* restrict c2 = c1 + ldc;
    double* restrict c3 = c2 + ldc;
    const double* b0 = B + (size_t)j * ldb;
    const double* b1 = b0 + ldb;
    const double* b2 = b1 + ldb;
    const double* b3 = b2 + ldb;
    int64_t k = 0;
    for (; k + 4 <= kc; k += 4) {
      const double* a0 = A + (size_t)k * lda;
      const double* a1 = a0 + lda;
      const double* a2 = a1 + lda;
      const double* a3 = a2 + lda;
      const double x00 = b0[k], x01 = b0[k + 1], x02 = b0[k + 2], x03 = b0[k + 3];
      const double x10 = b1[k], x11 = b1[k + 1], x12 = b1[k + 2], x13 = b1[k + 3];
      const double x20 = b2[k], x21 = b2[k + 1], x22 = b2[k + 2], x23 = b2[k + 3];
      const double x30 = b3[k], x31 = b3[k + 1], x32 = b3[k + 2], x33 = b3[k + 3];
      for (int64_t i = 0; i < mc; ++i) {
        const double p0 = a0[i], p1 = a1[i], p2 = a2[i], p3 = a3[i];
        c0[i] = (((c0[i] + p0 * x00) + p1 * x01) + p2 * x02) + p3 * x03;
        c1[i] = (((c1[i] + p0 * x10) + p1 * x11) + p2 * x12) + p3 * x13;
        c2[i] = (((c2[i] + p0 * x20) + p1 * x21) + p2 * x22) + p3 * x23;
        c3[i] = (((c3[i] + p0 * x30) + p1 * x31) + p2 * x32) + p3 * x33;
      }
    }
    for (; k < kc; ++k) {
      const double* a0 = A + (size_t)k * lda;
      const double x0 = b0[k], x1 = b1[k], x2 = b2[k], x3 = b3[k];
      for (int64_t i = 0; i < mc; ++i) {
        const double p = a0[i];
        c0[i] += p * x0;
        c1[i] += p * x1;
        c2[i] += p * x2;
        c3[i] += p * x3;
      }
    }
  }
  for (; j < nc; ++j) {
    double* restrict c = C + (size_t)j * ldc;
    const double* b = B + (size_t)j * ldb;
    int64_t k = 0;
    for (; k + 4 <= kc; k += 4) {
      const double* a0 = A + (size_t)k * lda;
      const double* a1 = a0 + lda;
      const double* a2 = a1 + lda;
      const double* a3 = a2 + lda;
      const double x0 = b[k], x1 = b[k + 1], x2 = b[k + 2], x3 = b[k + 3];
      for (int64_t i = 0; i < mc; ++i) c[i] = (((c[i] + a0[i] * x0) + a1[i] * x1) + a2[i] * x2) + a3[i] * x3;
    }
    for (; k < kc; ++k) {
      const double* a0 = A + (size_t)k * lda;
      const double x = b[k];
      for (int64_t i = 0; i < mc; ++i) c[i] += a0[i] * x;
    }
  }
}

/* C = A * B.  OpenMP over (row block, column block) tiles of C; each output
 * element is summed over k in ascending order from zero (gemm_block), so the
 * result does not depend on the thread count or the blocking. */
void lro_gemm_nn(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                 const double* B, int64_t ldb, double* C, int64_t ldc) {
  const int64_t NB = 16, MB = 512, KB = 256;
  const int64_t nj = (N + NB - 1) / NB, ni = (M + MB - 1) / MB;
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t jb = 0; jb < nj; ++jb)
    for (int64_t ib = 0; ib < ni; ++ib) {
      const int64_t j0 = jb * NB, j1 = j0 + NB < N ? j0 + NB : N;
      const int64_t i0 = ib * MB, i1 = i0 + MB < M ? i0 + MB : M;
      for (int64_t j = j0; j < j1; ++j)
        for (int64_t i = i0; i < i1; ++i) C[IDX(i, j, ldc)] = 0.0;
      for (int64_t k0 = 0; k0 < K; k0 += KB) {
        const int64_t k1 = k0 + KB < K ? k0 + KB : K;
        gemm_block(i1 - i0, j1 - j0, k1 - k0, A + IDX(i0, k0, lda), lda, B + IDX(k0, j0, ldb), ldb,
                   C + IDX(i0, j0, ldc), ldc);
      }
    }
}

/* C = A^T * B  (A is K x M) */
static void gemm_tn(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                    const double* B, int64_t ldb, double* C, int64_t ldc) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < N; ++j)
    for (int64_t i = 0; i < M; ++i) {
      double s = 0.0;
      const double* a = A + (size_t)i * lda;
      const double* b = B + (size_t)j * ldb;
      for (int64_t k = 0; k < K; ++k) s += a[k] * b[k];
      C[IDX(i, j, ldc)] = s;
    }
}

static void transpose(int64_t m, int64_t n, const double* a, int64_t lda, double* out /* n x m */) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) out[IDX(j, i, n)] = a[IDX(i, j, lda)];
}

/* -------------------------------------------------------------- cpqr.hpp */

/* cpqr.hpp:32-114: partial column-pivoted Householder QR stopped after k
 * steps.  Behaviour restated exactly:
 *  - pivot = first maximum of norm2 over positions [step, n) (strict >,
 *    cpqr.hpp:49-51), i.e. ties go to the lowest current position;
 *  - swap column, norm2, norm2_exact and pivot entries (cpqr.hpp:52-57);
 *  - reflector convention beta = -sign(alpha)|x|, tau = (beta-alpha)/beta,
 *    v = x/(alpha-beta) below the diagonal (cpqr.hpp:59-66);
 *  - trailing w = T^T v then T -= (tau v) w^T (cpqr.hpp:68-75);
 *  - downdate norm2 -= s_{step,j}^2 and recompute exactly once the value
 *    falls below 1e-6 x the last exact value (cpqr.hpp:78-84);
 *  - q = H_0..H_{k-1} [I;0] (cpqr.hpp:91-103) and the sign fix making
 *    diag(s) nonnegative (cpqr.hpp:105-112). */
int lro_cpqr(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
             double* q, double* s, int64_t* pivots, double* tau_out, int64_t* stats) {
  int rc;
  if ((rc = require_nonempty(m, n, "cpqr_partial"))) return rc;
  if ((rc = require_finite(m, n, a, lda, "cpqr_partial"))) return rc;
  if ((rc = require_rank_in_range(k, m, n, "cpqr_partial"))) return rc;

  double* work = NEW(double, m * n);
  double* tau = NEW(double, k);
  double* norm2 = NEW(double, n);
  double* norm2_exact = NEW(double, n);
  double* v = NEW(double, m);
  double* tv = NEW(double, m);
  double* w = NEW(double, n);
  if (!work || !tau || !norm2 || !norm2_exact || !v || !tv || !w) {
    free(work); free(tau); free(norm2); free(norm2_exact); free(v); free(tv); free(w);
    return fail(LRO_ENOMEM, "cpqr_partial: out of memory");
  }
  for (int64_t j = 0; j < n; ++j) memcpy(work + (size_t)j * m, a + (size_t)j * lda, sizeof(double) * m);
  for (int64_t j = 0; j < k; ++j) tau[j] = 0.0;
  for (int64_t j = 0; j < n; ++j) pivots[j] = j;
  for (int64_t j = 0; j < n; ++j) {
    double acc = 0.0;
    const double* c = work + (size_t)j * m;
    for (int64_t i = 0; i < m; ++i) acc += c[i] * c[i];
    norm2[j] = acc;
    norm2_exact[j] = acc;
  }
  int64_t recomputes = 0;

  for (int64_t step = 0; step < k; ++step) {
    int64_t pivot = step;
    for (int64_t j = step + 1; j < n; ++j)
      if (norm2[j] > norm2[pivot]) pivot = j;
    if (pivot != step) {
      double* cs = work + (size_t)step * m;
      double* cp = work + (size_t)pivot * m;
      for (int64_t i = 0; i < m; ++i) { double t = cs[i]; cs[i] = cp[i]; cp[i] = t; }
      double t = norm2[step]; norm2[step] = norm2[pivot]; norm2[pivot] = t;
      t = norm2_exact[step]; norm2_exact[step] = norm2_exact[pivot]; norm2_exact[pivot] = t;
      int64_t ti = pivots[step]; pivots[step] = pivots[pivot]; pivots[pivot] = ti;
    }

    const int64_t tail = m - step;
    double* col = work + (size_t)step * m;
    const double alpha = col[step];
    double cn2 = 0.0;
    for (int64_t i = step; i < m; ++i) cn2 += col[i] * col[i];
    const double colnorm = sqrt(cn2);
    if (colnorm > 0.0) {
      const double beta = alpha >= 0.0 ? -colnorm : colnorm;
      tau[step] = (beta - alpha) / beta;
      const double scale = alpha - beta;
      for (int64_t i = step + 1; i < m; ++i) col[i] /= scale;
      col[step] = beta;
      if (step + 1 < n) {
        v[0] = 1.0;
        for (int64_t i = 1; i < tail; ++i) v[i] = col[step + i];
        for (int64_t i = 0; i < tail; ++i) tv[i] = tau[step] * v[i];
        const int64_t nt = n - step - 1;
#pragma omp parallel for schedule(static) if (nt * tail > 262144)
        for (int64_t jj = 0; jj < nt; ++jj) {
          double* c = work + (size_t)(step + 1 + jj) * m + step;
          double acc = 0.0;
          for (int64_t i = 0; i < tail; ++i) acc += c[i] * v[i];
          for (int64_t i = 0; i < tail; ++i) c[i] -= tv[i] * acc;
        }
      }
    }

    for (int64_t j = step + 1; j < n; ++j) {
      const double sj = work[IDX(step, j, m)];
      norm2[j] -= sj * sj;
      if (norm2[j] < 1e-6 * norm2_exact[j]) {
        double acc = 0.0;
        const double* c = work + (size_t)j * m;
        for (int64_t i = step + 1; i < m; ++i) acc += c[i] * c[i];
        norm2[j] = acc;
        norm2_exact[j] = acc;
        ++recomputes;
      }
    }
  }

  int64_t* negative = NEW(int64_t, k);
  for (int64_t j = 0; j < k; ++j) negative[j] = work[IDX(j, j, m)] < 0.0;

  if (q) {
    /* cpqr.hpp:91-103 */
    for (int64_t j = 0; j < k; ++j)
      for (int64_t i = 0; i < m; ++i) q[IDX(i, j, m)] = (i == j) ? 1.0 : 0.0;
    for (int64_t step = k - 1; step >= 0; --step) {
      if (tau[step] == 0.0) continue;
      const int64_t tail = m - step;
      v[0] = 1.0;
      for (int64_t i = 1; i < tail; ++i) v[i] = work[IDX(step + i, step, m)];
      for (int64_t i = 0; i < tail; ++i) tv[i] = tau[step] * v[i];
      for (int64_t j = 0; j < k; ++j) {
        double* c = q + (size_t)j * m + step;
        double acc = 0.0;
        for (int64_t i = 0; i < tail; ++i) acc += c[i] * v[i];
        for (int64_t i = 0; i < tail; ++i) c[i] -= tv[i] * acc;
      }
    }
    for (int64_t j = 0; j < k; ++j)
      if (negative[j])
        for (int64_t i = 0; i < m; ++i) q[IDX(i, j, m)] = -q[IDX(i, j, m)];
  }
  /* cpqr.hpp:105-112 */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < k; ++i) {
      double val = (i > j) ? 0.0 : work[IDX(i, j, m)];
      if (negative[i]) val = -val;
      s[IDX(i, j, k)] = val;
    }
  if (tau_out) memcpy(tau_out, tau, sizeof(double) * k);
  if (stats) stats[0] = recomputes;
  free(negative); free(work); free(tau); free(norm2); free(norm2_exact); free(v); free(tv); free(w);
  return LRO_OK;
}

/* --------------------------------------------------------------- svd.hpp */

/* svd.hpp:39-93: one-sided Hestenes Jacobi on the columns of b (m >= n),
 * cyclic (p<q) order, tol 1e-14 relative, at most 60 sweeps; columns at the
 * eps^2 floor are zeroed.  Returns 1 on convergence. */
static int jacobi_orthogonalize_columns(int64_t m, int64_t n, double* b, double* v) {
  const double rel_tol = 1e-14;
  const int max_sweeps = 60;
  const double eps = 2.220446049250313e-16;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) v[IDX(i, j, n)] = (i == j) ? 1.0 : 0.0;
  double* norm2 = NEW(double, n);
  double* bp = NEW(double, m > n ? m : n);
  int converged = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    double mx = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      const double* c = b + (size_t)j * m;
      for (int64_t i = 0; i < m; ++i) acc += c[i] * c[i];
      norm2[j] = acc;
      if (j == 0 || acc > mx) mx = acc;
    }
    const double floor2 = mx * eps * eps;
#define DROP_IF_NEGLIGIBLE(jj)                                              \
  do {                                                                      \
    if (norm2[jj] <= floor2 && norm2[jj] != 0.0) {                          \
      for (int64_t i_ = 0; i_ < m; ++i_) b[IDX(i_, jj, m)] = 0.0;           \
      norm2[jj] = 0.0;                                                      \
    }                                                                       \
  } while (0)
    for (int64_t j = 0; j < n; ++j) DROP_IF_NEGLIGIBLE(j);

    double worst = 0.0;
    for (int64_t p = 0; p < n - 1; ++p) {
      for (int64_t qq = p + 1; qq < n; ++qq) {
        const double app = norm2[p], aqq = norm2[qq];
        if (app == 0.0 || aqq == 0.0) continue;
        double* cp = b + (size_t)p * m;
        double* cq = b + (size_t)qq * m;
        double apq = 0.0;
        for (int64_t i = 0; i < m; ++i) apq += cp[i] * cq[i];
        const double rel = fabs(apq) / sqrt(app * aqq);
        if (rel > worst) worst = rel;
        if (rel <= rel_tol) continue;
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        for (int64_t i = 0; i < m; ++i) {
          const double x = cp[i], y = cq[i];
          cp[i] = c * x - s * y;
          cq[i] = s * x + c * y;
        }
        double* vp = v + (size_t)p * n;
        double* vq = v + (size_t)qq * n;
        for (int64_t i = 0; i < n; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = c * x - s * y;
          vq[i] = s * x + c * y;
        }
        double np = c * c * app - 2.0 * c * s * apq + s * s * aqq;
        double nq = s * s * app + 2.0 * c * s * apq + c * c * aqq;
        norm2[p] = np > 0.0 ? np : 0.0;
        norm2[qq] = nq > 0.0 ? nq : 0.0;
        DROP_IF_NEGLIGIBLE(p);
        DROP_IF_NEGLIGIBLE(qq);
      }
    }
#undef DROP_IF_NEGLIGIBLE
    if (worst <= rel_tol) { converged = 1; break; }
  }
  free(norm2);
  free(bp);
  return converged;
}

/* svd.hpp:97-120: deterministic orthonormal completion of zero columns */
static void complete_basis(int64_t m, int64_t ncols, double* u, const int64_t* zero_cols, int64_t nz) {
  int64_t candidate = 0;
  double* e = NEW(double, m);
  for (int64_t zi = 0; zi < nz; ++zi) {
    const int64_t col = zero_cols[zi];
    for (; candidate < m; ++candidate) {
      for (int64_t i = 0; i < m; ++i) e[i] = 0.0;
      e[candidate] = 1.0;
      for (int64_t j = 0; j < ncols; ++j) {
        int pending = 0;
        for (int64_t t = 0; t < nz; ++t)
          if (zero_cols[t] == j) { pending = j >= col; break; }
        if (pending) continue;
        const double* uj = u + (size_t)j * m;
        double d = 0.0;
        for (int64_t i = 0; i < m; ++i) d += uj[i] * e[i];
        for (int64_t i = 0; i < m; ++i) e[i] -= d * uj[i];
      }
      double nrm = 0.0;
      for (int64_t i = 0; i < m; ++i) nrm += e[i] * e[i];
      nrm = sqrt(nrm);
      if (nrm > 0.5) {
        for (int64_t i = 0; i < m; ++i) u[IDX(i, col, m)] = e[i] / nrm;
        ++candidate;
        break;
      }
    }
  }
  free(e);
}

/* svd.hpp:132-183 */
int lro_svd(int64_t m, int64_t n, const double* a, int64_t lda, double* u, double* sigma, double* v) {
  int rc;
  if ((rc = require_nonempty(m, n, "svd"))) return rc;
  if ((rc = require_finite(m, n, a, lda, "svd"))) return rc;
  const int transposed = m < n;
  const int64_t bm = transposed ? n : m, bn = transposed ? m : n;
  double* b = NEW(double, bm * bn);
  double* vv = NEW(double, bn * bn);
  if (transposed) transpose(m, n, a, lda, b);
  else
    for (int64_t j = 0; j < n; ++j) memcpy(b + (size_t)j * m, a + (size_t)j * lda, sizeof(double) * m);
  if (!jacobi_orthogonalize_columns(bm, bn, b, vv)) {
    free(b); free(vv);
    return fail(LRO_ECONVERGE, "svd: one-sided Jacobi did not converge within 60 sweeps for %lldx%lld input",
                (long long)m, (long long)n);
  }
  double* sg = NEW(double, bn);
  for (int64_t j = 0; j < bn; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < bm; ++i) acc += b[IDX(i, j, bm)] * b[IDX(i, j, bm)];
    sg[j] = sqrt(acc);
  }
  /* stable descending sort (svd.hpp:155-158): insertion sort is stable */
  int64_t* order = NEW(int64_t, bn);
  for (int64_t j = 0; j < bn; ++j) order[j] = j;
  for (int64_t i = 1; i < bn; ++i) {
    int64_t x = order[i], j = i - 1;
    while (j >= 0 && sg[x] > sg[order[j]]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = x;
  }
  double* uu = NEW(double, bm * bn);   /* bm x bn */
  double* vo = NEW(double, bn * bn);   /* bn x bn */
  const double eps = 2.220446049250313e-16;
  const double zero_cutoff = sg[order[0]] * eps * (double)(bm > bn ? bm : bn);
  int64_t* zero_cols = NEW(int64_t, bn);
  int64_t nz = 0;
  for (int64_t j = 0; j < bn; ++j) {
    const int64_t src = order[j];
    sigma[j] = sg[src];
    memcpy(vo + (size_t)j * bn, vv + (size_t)src * bn, sizeof(double) * bn);
    if (sg[src] > zero_cutoff) {
      for (int64_t i = 0; i < bm; ++i) uu[IDX(i, j, bm)] = b[IDX(i, src, bm)] / sg[src];
    } else {
      for (int64_t i = 0; i < bm; ++i) uu[IDX(i, j, bm)] = 0.0;
      zero_cols[nz++] = j;
    }
  }
  if (nz) complete_basis(bm, bn, uu, zero_cols, nz);
  /* transposed: u <-> v (svd.hpp:181) */
  if (transposed) {
    memcpy(u, vo, sizeof(double) * bn * bn);   /* m x m */
    memcpy(v, uu, sizeof(double) * bm * bn);   /* n x m */
  } else {
    memcpy(u, uu, sizeof(double) * bm * bn);   /* m x n */
    memcpy(v, vo, sizeof(double) * bn * bn);   /* n x n */
  }
  free(b); free(vv); free(sg); free(order); free(uu); free(vo); free(zero_cols);
  return LRO_OK;
}

/* svd.hpp:193-207 and Svd::rank svd.hpp:22-27 */
int lro_pinv(int64_t m, int64_t n, const double* a, int64_t lda, double threshold, double* out) {
  if (!(threshold > 0.0 && threshold < 1.0))
    return fail(LRO_EINVAL, "pinv: threshold must lie in (0,1)");
  const int64_t r = m < n ? m : n;
  double* u = NEW(double, m * r);
  double* sg = NEW(double, r);
  double* v = NEW(double, n * r);
  int rc = lro_svd(m, n, a, lda, u, sg, v);
  if (rc) { free(u); free(sg); free(v); return rc; }
  int64_t rank = 0;
  if (sg[0] != 0.0)
    while (rank < r && sg[rank] >= threshold * sg[0]) ++rank;
  /* out (n x m) = (V_r diag(1/s)) U_r^T */
  for (int64_t l = 0; l < rank; ++l) {
    const double inv = 1.0 / sg[l];
    for (int64_t i = 0; i < n; ++i) v[IDX(i, l, n)] *= inv;
  }
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int64_t l = 0; l < rank; ++l) acc += v[IDX(i, l, n)] * u[IDX(j, l, m)];
      out[IDX(i, j, n)] = acc;
    }
  free(u); free(sg); free(v);
  return LRO_OK;
}

/* ------------------------------------------------------------- solve.hpp */

/* solve.hpp:39-60 */
static void conjugate_gradient(int64_t k, const double* normal, const double* rhs, double* x) {
  double* r = NEW(double, k);
  double* d = NEW(double, k);
  double* nd = NEW(double, k);
  double rho = 0.0, rhs2 = 0.0;
  for (int64_t i = 0; i < k; ++i) { x[i] = 0.0; r[i] = rhs[i]; d[i] = rhs[i]; rho += r[i] * r[i]; }
  rhs2 = rho;
  const double stop = 1e-28 * rhs2;
  const int64_t max_iters = 8 * k + 16;
  for (int64_t it = 0; it < max_iters && rho > stop; ++it) {
    for (int64_t i = 0; i < k; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < k; ++j) acc += normal[IDX(i, j, k)] * d[j];
      nd[i] = acc;
    }
    double denom = 0.0;
    for (int64_t i = 0; i < k; ++i) denom += d[i] * nd[i];
    if (denom <= 0.0) break;
    const double alpha = rho / denom;
    for (int64_t i = 0; i < k; ++i) x[i] += alpha * d[i];
    for (int64_t i = 0; i < k; ++i) r[i] -= alpha * nd[i];
    double rho_next = 0.0;
    for (int64_t i = 0; i < k; ++i) rho_next += r[i] * r[i];
    for (int64_t i = 0; i < k; ++i) d[i] = r[i] + (rho_next / rho) * d[i];
    rho = rho_next;
  }
  free(r); free(d); free(nd);
}

/* solve.hpp:62-89: row-oriented back substitution */
static int back_substitute(int64_t k, int64_t nc, const double* s11, int64_t ld11, const double* s12,
                           int64_t ld12, double threshold, int allow_singularity_error, double* t) {
  double diag_max = 0.0;
  for (int64_t i = 0; i < k; ++i) {
    const double d = fabs(s11[IDX(i, i, ld11)]);
    if (i == 0 || d > diag_max) diag_max = d;
  }
  const double diag_tol = threshold * diag_max;
  double rhs_scale = 0.0;
  for (int64_t j = 0; j < nc; ++j)
    for (int64_t i = 0; i < k; ++i) {
      const double x = fabs(s12[IDX(i, j, ld12)]);
      if (x > rhs_scale) rhs_scale = x;
    }
  int rc = LRO_OK;
  int64_t bad = -1;
  for (int64_t i = k - 1; i >= 0; --i) {
    const double dii = s11[IDX(i, i, ld11)];
    const int zero_row = fabs(dii) <= diag_tol;
    double residual = 0.0;
#pragma omp parallel for schedule(static) reduction(max : residual) if (nc > 4096)
    for (int64_t c = 0; c < nc; ++c) {
      double rhs = s12[IDX(i, c, ld12)];
      for (int64_t j = i + 1; j < k; ++j) rhs -= s11[IDX(i, j, ld11)] * t[IDX(j, c, k)];
      if (zero_row) {
        if (fabs(rhs) > residual) residual = fabs(rhs);
        t[IDX(i, c, k)] = 0.0;
      } else {
        t[IDX(i, c, k)] = rhs / dii;
      }
    }
    if (zero_row && allow_singularity_error && residual > threshold * rhs_scale) {
      bad = i;
      rc = LRO_ESINGULAR;
      break;
    }
  }
  if (rc) {
    g_sing_index = bad;
    return fail(LRO_ESINGULAR,
                "stabilized_coeff_solve: zero diagonal with inconsistent right-hand side at index %lld",
                (long long)bad);
  }
  return LRO_OK;
}

/* solve.hpp:104-145 */
int lro_coeff_solve(int64_t k, int64_t nc, const double* s11, int64_t ld11, const double* s12,
                    int64_t ld12, lro_solve_strategy strat, double* t) {
  if (k < 0 || nc < 0) return fail(LRO_EINVAL, "stabilized_coeff_solve: row count mismatch");
  if (!all_finite(k, k, s11, ld11) || !all_finite(k, nc, s12, ld12))
    return fail(LRO_EINVAL, "stabilized_coeff_solve: non-finite entries");
  for (int64_t j = 0; j < k; ++j)
    for (int64_t i = j + 1; i < k; ++i)
      if (s11[IDX(i, j, ld11)] != 0.0)
        return fail(LRO_EINVAL, "stabilized_coeff_solve: block is not upper triangular");
  if (nc == 0) return LRO_OK;

  int kind = strat.kind;
  if (kind == LRO_SOLVE_BACKSUB && strat.escalate) {
    double dmax = 0.0, dmin = 0.0;
    for (int64_t i = 0; i < k; ++i) {
      const double d = fabs(s11[IDX(i, i, ld11)]);
      if (i == 0 || d > dmax) dmax = d;
      if (i == 0 || d < dmin) dmin = d;
    }
    if (dmax == 0.0 || dmin == 0.0 || dmax / dmin > 1e10) kind = LRO_SOLVE_PINV;
  }
  switch (kind) {
    case LRO_SOLVE_BACKSUB:
      return back_substitute(k, nc, s11, ld11, s12, ld12, strat.threshold, !strat.escalate, t);
    case LRO_SOLVE_PINV: {
      double* p = NEW(double, k * k);
      int rc = lro_pinv(k, k, s11, ld11, strat.threshold, p);
      if (rc) { free(p); return rc; }
      /* pinv(s11) * s12 */
      double* s12c = NEW(double, k * nc);
      for (int64_t j = 0; j < nc; ++j) memcpy(s12c + (size_t)j * k, s12 + (size_t)j * ld12, sizeof(double) * k);
      lro_gemm_nn(k, nc, k, p, k, s12c, k, t, k);
      free(p); free(s12c);
      return LRO_OK;
    }
    case LRO_SOLVE_TIKHONOV: {
      const double ridge2 = strat.ridge * strat.ridge;
      double* normal = NEW(double, k * k);
      for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < k; ++i) {
          double acc = 0.0;
          for (int64_t l = 0; l < k; ++l) acc += s11[IDX(l, i, ld11)] * s11[IDX(l, j, ld11)];
          normal[IDX(i, j, k)] = acc + (i == j ? ridge2 : 0.0);
        }
      double* rhs = NEW(double, k);
      for (int64_t c = 0; c < nc; ++c) {
        for (int64_t i = 0; i < k; ++i) {
          double acc = 0.0;
          for (int64_t l = 0; l < k; ++l) acc += s11[IDX(l, i, ld11)] * s12[IDX(l, c, ld12)];
          rhs[i] = acc;
        }
        conjugate_gradient(k, normal, rhs, t + (size_t)c * k);
      }
      free(normal); free(rhs);
      return LRO_OK;
    }
  }
  return fail(LRO_ERUNTIME, "stabilized_coeff_solve: unreachable");
}

/* ---------------------------------------------------------------- id.hpp */

/* id.hpp:91-105 */
int lro_id_column(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                  lro_solve_strategy strat, int64_t* pivots, double* coeff) {
  int rc;
  if ((rc = require_rank_in_range(k, m, n, "id_column"))) return rc;
  double* s = NEW(double, k * n);
  rc = lro_cpqr(m, n, a, lda, k, NULL, s, pivots, NULL, NULL);
  if (!rc) rc = lro_coeff_solve(k, n - k, s, k, s + (size_t)k * k, k, strat, coeff);
  free(s);
  return rc;
}

/* id.hpp:108-119: column ID of the transpose */
int lro_id_row(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
               lro_solve_strategy strat, int64_t* pivots, double* coeff) {
  int rc;
  if ((rc = require_rank_in_range(k, n, m, "id_column"))) return rc;
  double* at = NEW(double, m * n);
  transpose(m, n, a, lda, at);
  rc = lro_id_column(n, m, at, n, k, strat, pivots, coeff);
  free(at);
  return rc;
}

/* ------------------------------------------------------------ sketch.hpp */

/* sketch.hpp:54-58 */
static int require_sample_count(int64_t ell, int64_t rows, const char* who) {
  if (ell < 1 || ell > rows)
    return fail(LRO_EINVAL, "%s: sample count %lld out of range for %lld rows", who, (long long)ell,
                (long long)rows);
  return LRO_OK;
}

/* sketch.hpp:67-78 */
int lro_sketch_gaussian(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell,
                        uint64_t seed, double* y) {
  int rc;
  if ((rc = require_nonempty(m, n, "sketch_gaussian"))) return rc;
  if ((rc = require_finite(m, n, a, lda, "sketch_gaussian"))) return rc;
  if ((rc = require_sample_count(ell, m, "sketch_gaussian"))) return rc;
  double* omega = NEW(double, ell * m);
  if (!omega) return fail(LRO_ENOMEM, "sketch_gaussian: out of memory");
  lro_gaussian_matrix(ell, m, seed, omega);
  lro_gemm_nn(ell, n, m, omega, ell, a, lda, y, ell);
  free(omega);
  return LRO_OK;
}

/* sketch.hpp:200-223 with build_sample (sketch.hpp:169-189) at q = 0 */
int lro_randomized_id(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int oversample,
                      uint64_t seed, lro_solve_strategy strat, int64_t* pivots, double* coeff,
                      int64_t* stats) {
  int rc;
  if ((rc = require_rank_in_range(k, m, n, "randomized_id"))) return rc;
  const int64_t ell = k + (int64_t)oversample; /* SketchConfig::sample_count, sketch.hpp:29-32 */
  if (ell < k) return fail(LRO_EINVAL, "build_sample: sample count below target rank");
  double* y = NEW(double, ell * n);
  if ((rc = lro_sketch_gaussian(m, n, a, lda, ell, seed, y))) { free(y); return rc; }
  const int64_t steps = ell < n ? ell : n; /* cpqr_full, cpqr.hpp:118-122 */
  if (steps < k) { free(y); return fail(LRO_ERUNTIME, "randomized_id: sample rank collapsed below target rank"); }
  double* s = NEW(double, steps * n);
  rc = lro_cpqr(ell, n, y, ell, steps, NULL, s, pivots, NULL, stats);
  if (!rc) {
    /* s1 = top k rows (sketch.hpp:213-215) */
    double* s1 = NEW(double, k * n);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < k; ++i) s1[IDX(i, j, k)] = s[IDX(i, j, steps)];
    rc = lro_coeff_solve(k, n - k, s1, k, s1 + (size_t)k * k, k, strat, coeff);
    free(s1);
  }
  free(s); free(y);
  return rc;
}

static const double kPi = 3.14159265358979323846; /* std::numbers::pi */

/* rng.hpp:53-62 */
void lro_sample_without_replacement(uint64_t seed, int64_t population, int64_t count, int64_t* out) {
  int64_t* pool = NEW(int64_t, population);
  for (int64_t i = 0; i < population; ++i) pool[i] = i;
  uint64_t next = 0;
  for (int64_t i = 0; i < count; ++i) {
    const int64_t j = i + (int64_t)(lro_stream_value(seed, next++) % (uint64_t)(population - i));
    const int64_t t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
  }
  memcpy(out, pool, sizeof(int64_t) * (size_t)count);
  free(pool);
}

static double srft_sign(uint64_t sign_seed, int64_t i) {
  return (lro_stream_value(sign_seed, (uint64_t)i) & 1u) ? -1.0 : 1.0;
}

/* sketch.hpp:84-100 with hartley.hpp:60-73 */
int lro_srft_operator(int64_t m, int64_t ell, uint64_t seed, double* out) {
  if (ell < 1 || ell > m) return fail(LRO_EINVAL, "srft_operator: sample count %lld out of range for %lld rows",
                                      (long long)ell, (long long)m);
  const uint64_t sseed = lro_derive_seed(seed, 1), rseed = lro_derive_seed(seed, 2);
  int64_t* rows = NEW(int64_t, ell);
  lro_sample_without_replacement(rseed, m, ell, rows);
  const double hs = 1.0 / sqrt((double)m), scale = sqrt((double)m / (double)ell);
  for (int64_t q = 0; q < m; ++q) {
    const double sg = srft_sign(sseed, q);
    for (int64_t i = 0; i < ell; ++i) {
      const int64_t p = rows[i];
      const double t = 2.0 * kPi * (double)((p * q) % m) / (double)m;
      out[IDX(i, q, ell)] = scale * ((hs * (cos(t) + sin(t))) * sg);
    }
  }
  free(rows);
  return LRO_OK;
}

/* hartley.hpp:17-43: unnormalised radix-2 DIT fast Hartley transform */
static void fht_unnormalized(double* data, double* scratch, int64_t n) {
  if (n == 1) return;
  const int64_t half = n / 2;
  for (int64_t j = 0; j < half; ++j) {
    scratch[j] = data[2 * j];
    scratch[half + j] = data[2 * j + 1];
  }
  fht_unnormalized(scratch, data, half);
  fht_unnormalized(scratch + half, data, half);
  const double* even = scratch;
  const double* odd = scratch + half;
  for (int64_t k = 0; k < half; ++k) {
    const double angle = 2.0 * kPi * (double)k / (double)n;
    const double c = cos(angle), s = sin(angle);
    const int64_t mirror = k == 0 ? 0 : half - k;
    const double cross = c * odd[k] + s * odd[mirror];
    data[k] = even[k] + cross;
    data[k + half] = even[k] - cross;
  }
}

/* sketch.hpp:110-143 */
int lro_sketch_srft(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, uint64_t seed, double* y) {
  if (m < 1 || n < 1) return fail(LRO_EINVAL, "sketch_srft: matrix must be nonempty");
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i)
      if (!isfinite(a[IDX(i, j, lda)])) return fail(LRO_EINVAL, "sketch_srft: matrix has non-finite entries");
  if (ell < 1 || ell > m) return fail(LRO_EINVAL, "sketch_srft: sample count %lld out of range for %lld rows",
                                      (long long)ell, (long long)m);
  if ((m & (m - 1)) == 0) {
    const uint64_t sseed = lro_derive_seed(seed, 1), rseed = lro_derive_seed(seed, 2);
    int64_t* rows = NEW(int64_t, ell);
    lro_sample_without_replacement(rseed, m, ell, rows);
    double* col = NEW(double, m);
    double* scr = NEW(double, m);
    const double hs = 1.0 / sqrt((double)m), scale = sqrt((double)m / (double)ell);
    for (int64_t j = 0; j < n; ++j) {
      for (int64_t i = 0; i < m; ++i) col[i] = srft_sign(sseed, i) * a[IDX(i, j, lda)];
      fht_unnormalized(col, scr, m);
      for (int64_t i = 0; i < m; ++i) col[i] *= hs;
      for (int64_t i = 0; i < ell; ++i) y[IDX(i, j, ell)] = scale * col[rows[i]];
    }
    free(scr); free(col); free(rows);
    return LRO_OK;
  }
  double* om = NEW(double, ell * m);
  int rc = lro_srft_operator(m, ell, seed, om);
  if (!rc) lro_gemm_nn(ell, n, m, om, ell, a, lda, y, ell);
  free(om);
  return rc;
}

/* svd.hpp:216-235.  Eigen's HouseholderQR on y^T with makeHouseholder's
 * convention (beta = -sign(c0)|x|, tau = (beta - c0)/beta, v = x/(c0 - beta);
 * no reflection when the tail is exactly zero), then householderQ() applied to
 * the first r columns of the identity. */
int lro_orth_rows(int64_t ell, int64_t n, const double* y, int64_t ldy, double* out, int64_t* r_out) {
  if (ell < 1 || n < 1) return fail(LRO_EINVAL, "orth_rows: matrix must be nonempty");
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < ell; ++i)
      if (!isfinite(y[IDX(i, j, ldy)])) return fail(LRO_EINVAL, "orth_rows: matrix has non-finite entries");
  const int64_t rows = n, cols = ell, rmax = n < ell ? n : ell;
  double* x = NEW(double, rows * cols); /* x = y^T, rows x cols */
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) x[IDX(i, j, rows)] = y[IDX(j, i, ldy)];
  double* tau = NEW(double, rmax);
  double* diag = NEW(double, rmax);
  for (int64_t j = 0; j < rmax; ++j) {
    double* cj = x + (size_t)j * rows;
    const double c0 = cj[j];
    double tail = 0.0;
    for (int64_t i = j + 1; i < rows; ++i) tail += cj[i] * cj[i];
    double beta, t;
    if (tail == 0.0) {
      t = 0.0;
      beta = c0;
      for (int64_t i = j + 1; i < rows; ++i) cj[i] = 0.0;
    } else {
      beta = sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      for (int64_t i = j + 1; i < rows; ++i) cj[i] /= (c0 - beta);
      t = (beta - c0) / beta;
    }
    tau[j] = t;
    diag[j] = fabs(beta);
    cj[j] = beta;
    /* apply H = I - t v v^T (v_j = 1) to the trailing columns */
    for (int64_t c = j + 1; c < cols; ++c) {
      double* cc = x + (size_t)c * rows;
      double w = cc[j];
      for (int64_t i = j + 1; i < rows; ++i) w += cj[i] * cc[i];
      w *= t;
      cc[j] -= w;
      for (int64_t i = j + 1; i < rows; ++i) cc[i] -= w * cj[i];
    }
  }
  double dmax = 0.0;
  for (int64_t j = 0; j < rmax; ++j) dmax = diag[j] > dmax ? diag[j] : dmax;
  const double tol = dmax * DBL_EPSILON * (double)(rows > cols ? rows : cols);
  int64_t r = rmax;
  while (r > 0 && diag[r - 1] <= tol) --r;
  /* thin Q (rows x r) = H_0 ... H_{rmax-1} [I_r; 0] */
  double* q = NEW(double, rows * (r > 0 ? r : 1));
  for (int64_t c = 0; c < r; ++c)
    for (int64_t i = 0; i < rows; ++i) q[IDX(i, c, rows)] = (i == c) ? 1.0 : 0.0;
  for (int64_t j = rmax - 1; j >= 0; --j) {
    const double* vj = x + (size_t)j * rows;
    if (tau[j] == 0.0) continue;
    for (int64_t c = 0; c < r; ++c) {
      double* qc = q + (size_t)c * rows;
      double w = qc[j];
      for (int64_t i = j + 1; i < rows; ++i) w += vj[i] * qc[i];
      w *= tau[j];
      qc[j] -= w;
      for (int64_t i = j + 1; i < rows; ++i) qc[i] -= w * vj[i];
    }
  }
  for (int64_t c = 0; c < r; ++c)
    for (int64_t i = 0; i < rows; ++i) out[IDX(c, i, ldy)] = q[IDX(i, c, rows)];
  *r_out = r;
  free(q); free(diag); free(tau); free(x);
  return LRO_OK;
}

/* sketch.hpp:148-164 */
static int power_rounds(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, int q, int reorth,
                        double* y, int64_t* rows_out);

int lro_sketch_power(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, int q, int reorth,
                     uint64_t seed, double* y, int64_t* rows_out) {
  if (q < 0) return fail(LRO_EINVAL, "sketch_power: q must be nonnegative");
  int rc = lro_sketch_gaussian(m, n, a, lda, ell, seed, y);
  if (rc) return rc;
  return power_rounds(m, n, a, lda, ell, q, reorth, y, rows_out);
}

/* the power rounds of sketch_power / build_sample (sketch.hpp:155-160, :180-185) */
static int power_rounds(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, int q, int reorth,
                        double* y, int64_t* rows_out) {
  int rc = 0;
  int64_t rows = ell;
  if (q == 0) {
    *rows_out = ell;
    return 0;
  }
  double* z = NEW(double, ell * m);   /* ell x m, ld ell */
  double* at = NEW(double, n * m);    /* A^T, n x m */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) at[IDX(j, i, n)] = a[IDX(i, j, lda)];
  for (int round = 0; round < q && !rc; ++round) {
    if (reorth && (rc = lro_orth_rows(rows, n, y, ell, y, &rows))) break;
    lro_gemm_nn(rows, m, n, y, ell, at, n, z, ell);  /* z = y A^T */
    if (reorth && (rc = lro_orth_rows(rows, m, z, ell, z, &rows))) break;
    lro_gemm_nn(rows, n, m, z, ell, a, lda, y, ell);  /* y = z A */
  }
  free(at); free(z);
  *rows_out = rows;
  return rc;
}

int lro_randomized_id_power(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int oversample,
                            int q, int reorth, uint64_t seed, lro_solve_strategy strat, int64_t* pivots,
                            double* coeff, int64_t* stats) {
  return lro_randomized_id_cfg(m, n, a, lda, k, 0, oversample, 0, q, reorth, seed, strat, pivots, coeff, stats);
}

int lro_randomized_id_cfg(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int kind, int oversample,
                          int64_t srft_samples, int q, int reorth, uint64_t seed, lro_solve_strategy strat,
                          int64_t* pivots, double* coeff, int64_t* stats) {
  int rc;
  if ((rc = require_rank_in_range(k, m, n, "randomized_id"))) return rc;
  /* SketchConfig::sample_count, sketch.hpp:29-32 */
  const int64_t ell = kind == 0 ? k + (int64_t)oversample : (srft_samples > 0 ? srft_samples : 2 * k);
  if (ell < k) return fail(LRO_EINVAL, "build_sample: sample count below target rank");
  if (q < 0) return fail(LRO_EINVAL, "sketch_power: q must be nonnegative");
  double* y = NEW(double, ell * n);
  int64_t rows = ell;
  rc = kind == 0 ? lro_sketch_gaussian(m, n, a, lda, ell, seed, y) : lro_sketch_srft(m, n, a, lda, ell, seed, y);
  if (!rc) rc = power_rounds(m, n, a, lda, ell, q, reorth, y, &rows);
  if (rc) { free(y); return rc; }
  const int64_t steps = rows < n ? rows : n;
  if (steps < k) { free(y); return fail(LRO_ERUNTIME, "randomized_id: sample rank collapsed below target rank"); }
  double* s = NEW(double, steps * n);
  rc = lro_cpqr(rows, n, y, ell, steps, NULL, s, pivots, NULL, stats);
  if (!rc) {
    double* s1 = NEW(double, k * n);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < k; ++i) s1[IDX(i, j, k)] = s[IDX(i, j, steps)];
    rc = lro_coeff_solve(k, n - k, s1, k, s1 + (size_t)k * k, k, strat, coeff);
    free(s1);
  }
  free(s); free(y);
  return rc;
}

/* sketch.hpp:238-254 */
int lro_randomized_svd(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int kind, int oversample,
                       int64_t srft_samples, int q, int reorth, uint64_t seed, double* u, double* sigma, double* v) {
  int rc;
  if ((rc = require_rank_in_range(k, m, n, "randomized_svd"))) return rc;
  const int64_t ell = kind == 0 ? k + (int64_t)oversample : (srft_samples > 0 ? srft_samples : 2 * k);
  if (ell < k) return fail(LRO_EINVAL, "build_sample: sample count below target rank");
  double* y = NEW(double, ell * n);
  int64_t rows = ell, r = 0;
  rc = kind == 0 ? lro_sketch_gaussian(m, n, a, lda, ell, seed, y) : lro_sketch_srft(m, n, a, lda, ell, seed, y);
  if (!rc) rc = power_rounds(m, n, a, lda, ell, q, reorth, y, &rows);
  if (!rc) rc = lro_orth_rows(rows, n, y, ell, y, &r);  /* q (r x n, ld ell) */
  if (!rc && r < k) rc = fail(LRO_ERUNTIME, "randomized_svd: sample rank collapsed below target rank");
  if (rc) { free(y); return rc; }
  /* projected = a q^T (m x r) */
  double* qt = NEW(double, n * r);
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < n; ++j) qt[IDX(j, i, n)] = y[IDX(i, j, ell)];
  double* pr = NEW(double, m * r);
  lro_gemm_nn(m, r, n, a, lda, qt, n, pr, m);
  const int64_t rr = m < r ? m : r;
  double* su = NEW(double, m * rr);
  double* ss = NEW(double, rr);
  double* sv = NEW(double, r * rr);
  rc = lro_svd(m, r, pr, m, su, ss, sv);
  if (!rc) {
    memcpy(u, su, sizeof(double) * (size_t)(m * k));
    memcpy(sigma, ss, sizeof(double) * (size_t)k);
    lro_gemm_nn(n, k, r, qt, n, sv, r, v, n);  /* v = q^T small.v(:, :k) */
  }
  free(sv); free(ss); free(su); free(pr); free(qt); free(y);
  return rc;
}

/* id.hpp:124-134 */
int lro_tsid_from_column_id(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                            const int64_t* col_pivots, lro_solve_strategy strat, int64_t* row_pivots,
                            double* row_coeff, double* skeleton) {
  (void)n;
  double* c = NEW(double, m * k);
  for (int64_t j = 0; j < k; ++j) memcpy(c + (size_t)j * m, a + (size_t)col_pivots[j] * lda, sizeof(double) * m);
  int rc = lro_id_row(m, k, c, m, k, strat, row_pivots, row_coeff);
  if (!rc && skeleton)
    for (int64_t j = 0; j < k; ++j)
      for (int64_t i = 0; i < k; ++i) skeleton[IDX(i, j, k)] = c[IDX(row_pivots[i], j, m)];
  free(c);
  return rc;
}

/* --------------------------------------------------------------- cur.hpp */

/* cur.hpp:23-34 and lowrank_main.cpp:210-215 */
int lro_cur_from_two_sided(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                           const int64_t* col_pivots, const double* col_coeff,
                           const int64_t* row_pivots, double pinv_threshold, int u_mode, double* c,
                           double* u, double* r) {
  /* core.hpp:70-85 gathers */
  for (int64_t j = 0; j < k; ++j) memcpy(c + (size_t)j * m, a + (size_t)col_pivots[j] * lda, sizeof(double) * m);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < k; ++i) r[IDX(i, j, k)] = a[IDX(row_pivots[i], j, lda)];
  double* rp = NEW(double, n * k); /* pinv(r): n x k */
  int rc = lro_pinv(k, n, r, k, pinv_threshold, rp);
  if (rc) { free(rp); return rc; }
  if (u_mode == LRO_U_VT_RPINV) {
    /* u = basis()^T pinv(r); basis() is n x k (id.hpp:21-30) */
    double* basis = NEW(double, n * k);
    memset(basis, 0, sizeof(double) * n * k);
    for (int64_t l = 0; l < n; ++l) {
      if (l < k) basis[IDX(col_pivots[l], l, n)] = 1.0;
      else
        for (int64_t t = 0; t < k; ++t) basis[IDX(col_pivots[l], t, n)] = col_coeff[IDX(t, l - k, k)];
    }
    gemm_tn(k, k, n, basis, n, rp, n, u, k);
    free(basis);
  } else {
    double* cp = NEW(double, k * m); /* pinv(c): k x m */
    rc = lro_pinv(m, k, c, m, pinv_threshold, cp);
    if (rc) { free(cp); free(rp); return rc; }
    double* ca = NEW(double, k * n);
    lro_gemm_nn(k, n, m, cp, k, a, lda, ca, k);
    lro_gemm_nn(k, k, n, ca, k, rp, n, u, k);
    free(cp); free(ca);
  }
  free(rp);
  return LRO_OK;
}

/* core.hpp:64-67 on cur.hpp:77-80: ||A - (C U) R||_F and ||A||_F */
int lro_cur_error_fro(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, const double* c,
                      const double* u, const double* r, double* out) {
  double* cu = NEW(double, m * k);
  lro_gemm_nn(m, k, k, c, m, u, k, cu, m);
  /* (C U) R one 16-column block at a time (each entry summed over l
   * ascending, as gemm_block does); per-block partial sums are added in
   * block order, so the result does not depend on the thread count */
  const int64_t NB = 16, MB = 512, KB = 256;
  const int64_t nb = (n + NB - 1) / NB;
  double* part = NEW(double, 2 * nb);
#pragma omp parallel
  {
    double* p = NEW(double, MB * NB);
#pragma omp for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t j0 = b * NB, nc = j0 + NB < n ? NB : n - j0;
      double e2 = 0.0, x2 = 0.0;
      for (int64_t i0 = 0; i0 < m; i0 += MB) {
        const int64_t mc = i0 + MB < m ? MB : m - i0;
        for (int64_t t = 0; t < MB * NB; ++t) p[t] = 0.0;
        for (int64_t l0 = 0; l0 < k; l0 += KB)
          gemm_block(mc, nc, l0 + KB < k ? KB : k - l0, cu + IDX(i0, l0, m), m, r + IDX(l0, j0, k), k, p, MB);
        for (int64_t j = 0; j < nc; ++j)
          for (int64_t i = 0; i < mc; ++i) {
            const double x = a[IDX(i0 + i, j0 + j, lda)];
            const double d = x - p[IDX(i, j, MB)];
            e2 += d * d;
            x2 += x * x;
          }
      }
      part[2 * b] = e2;
      part[2 * b + 1] = x2;
    }
    free(p);
  }
  double err2 = 0.0, a2 = 0.0;
  for (int64_t b = 0; b < nb; ++b) {
    err2 += part[2 * b];
    a2 += part[2 * b + 1];
  }
  out[0] = sqrt(err2);
  out[1] = sqrt(a2);
  free(part);
  free(cu);
  return LRO_OK;
}
