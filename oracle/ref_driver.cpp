// ref_driver.cpp -- TEST-ONLY C-ABI driver over the UNMODIFIED reference
// headers (/root/reference/proj/include/lowrank), compiled in place against
// oracle/eigen_subset (Eigen 3.4 is absent from this image).  Built into
// oracle/_ref/liblowrank_ref.so by oracle/Makefile; it exists to pin the C
// restatement (lowrank_oracle.c) and, via bench.py --impl reference, to time
// the reference's own algorithm on the host.  Nothing here is product code.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "lowrank/lowrank.hpp"

using namespace lowrank;
using Mat = MatrixX<double>;

namespace {
thread_local std::string g_err;
thread_local int64_t g_sing = -1;

Mat from_ptr(int64_t m, int64_t n, const double* a, int64_t lda) {
  Mat out(m, n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) out(i, j) = a[i + j * lda];
  return out;
}
void to_ptr(const Mat& x, double* out) {
  for (Index j = 0; j < x.cols(); ++j)
    for (Index i = 0; i < x.rows(); ++i) out[i + j * x.rows()] = x(i, j);
}
void to_idx(const IndexVector& p, int64_t* out) {
  for (Index i = 0; i < p.size(); ++i) out[i] = p(i);
}
IndexVector from_idx(int64_t n, const int64_t* p) {
  IndexVector out(n);
  for (int64_t i = 0; i < n; ++i) out(i) = p[i];
  return out;
}
SolveStrategy strategy(int kind, double thr, double ridge, int escalate) {
  SolveStrategy s;
  s.kind = kind == 0 ? SolveKind::BackSubstitution : kind == 1 ? SolveKind::TruncatedPinv : SolveKind::Tikhonov;
  s.threshold = thr;
  s.ridge = ridge;
  s.escalate = escalate != 0;
  return s;
}
template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const SingularityError& e) {
    g_err = e.what();
    g_sing = e.index();
    return 2;
  } catch (const ConvergenceError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}
}  // namespace

extern "C" {

const char* lref_last_error() { return g_err.c_str(); }
int64_t lref_last_singular_index() { return g_sing; }

int lref_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  return guard([&] { to_ptr(gaussian_matrix<double>(rows, cols, seed), out); });
}

int lref_sketch_gaussian(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, uint64_t seed,
                         double* y) {
  return guard([&] { to_ptr(sketch_gaussian(from_ptr(m, n, a, lda), ell, seed).y, y); });
}

int lref_cpqr(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, double* q, double* s,
              int64_t* pivots) {
  return guard([&] {
    auto qr = cpqr_partial(from_ptr(m, n, a, lda), k);
    if (q) to_ptr(qr.q, q);
    to_ptr(qr.s, s);
    to_idx(qr.pivots, pivots);
  });
}

int lref_coeff_solve(int64_t k, int64_t nc, const double* s11, int64_t ld11, const double* s12, int64_t ld12,
                     int kind, double thr, double ridge, int escalate, double* t) {
  return guard([&] {
    to_ptr(stabilized_coeff_solve(from_ptr(k, k, s11, ld11), from_ptr(k, nc, s12, ld12),
                                  strategy(kind, thr, ridge, escalate)),
           t);
  });
}

int lref_svd(int64_t m, int64_t n, const double* a, int64_t lda, double* u, double* sigma, double* v) {
  return guard([&] {
    auto f = svd(from_ptr(m, n, a, lda));
    to_ptr(f.u, u);
    to_ptr(Mat(f.sigma), sigma);
    to_ptr(f.v, v);
  });
}

int lref_pinv(int64_t m, int64_t n, const double* a, int64_t lda, double thr, double* out) {
  return guard([&] { to_ptr(pinv(from_ptr(m, n, a, lda), thr), out); });
}

int lref_id_column(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int64_t* pivots,
                   double* coeff) {
  return guard([&] {
    auto id = id_column(from_ptr(m, n, a, lda), k);
    to_idx(id.pivots, pivots);
    to_ptr(id.coeff, coeff);
  });
}

int lref_id_row(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int64_t* pivots,
                double* coeff) {
  return guard([&] {
    auto id = id_row(from_ptr(m, n, a, lda), k);
    to_idx(id.pivots, pivots);
    to_ptr(id.coeff, coeff);
  });
}

int lref_randomized_id(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int oversample,
                       uint64_t seed, int64_t* pivots, double* coeff) {
  return guard([&] {
    SketchConfig cfg;
    cfg.oversample = oversample;
    cfg.seed = seed;
    auto id = randomized_id(from_ptr(m, n, a, lda), k, cfg);
    to_idx(id.pivots, pivots);
    to_ptr(id.coeff, coeff);
  });
}

// sketch.hpp:148-164 power sketch: y (ell x n, ld ell); *rows = final row count
int lref_sketch_power(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, int q, int reorth,
                      uint64_t seed, double* y, int64_t* rows) {
  return guard([&] {
    auto out = sketch_power(from_ptr(m, n, a, lda), ell, q, reorth != 0, seed);
    *rows = out.y.rows();
    for (int64_t j = 0; j < out.y.cols(); ++j)
      for (int64_t i = 0; i < out.y.rows(); ++i) y[i + j * ell] = out.y(i, j);
  });
}

// sketch.hpp:110-143: y (ell x n, ld ell)
int lref_sketch_srft(int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, uint64_t seed, double* y) {
  return guard([&] { to_ptr(sketch_srft(from_ptr(m, n, a, lda), ell, seed).y, y); });
}

int lref_srft_operator(int64_t m, int64_t ell, uint64_t seed, double* out) {
  return guard([&] { to_ptr(srft_operator<double>(m, ell, seed), out); });
}

// sketch.hpp:238-254
int lref_randomized_svd(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int kind, int oversample,
                        int64_t srft_samples, int q, int reorth, uint64_t seed, double* u, double* sigma, double* v) {
  return guard([&] {
    SketchConfig cfg;
    cfg.kind = kind == 0 ? SketchKind::Gaussian : SketchKind::Srft;
    cfg.oversample = oversample;
    cfg.srft_samples = srft_samples;
    cfg.seed = seed;
    cfg.power = q;
    cfg.reorthonormalize = reorth != 0;
    auto s = randomized_svd(from_ptr(m, n, a, lda), k, cfg);
    to_ptr(s.u, u);
    for (int64_t i = 0; i < k; ++i) sigma[i] = s.sigma(i);
    to_ptr(s.v, v);
  });
}

// sketch.hpp:200-223 with a full SketchConfig
int lref_randomized_id_cfg(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int kind, int oversample,
                           int64_t srft_samples, int q, int reorth, uint64_t seed, int64_t* pivots, double* coeff) {
  return guard([&] {
    SketchConfig cfg;
    cfg.kind = kind == 0 ? SketchKind::Gaussian : SketchKind::Srft;
    cfg.oversample = oversample;
    cfg.srft_samples = srft_samples;
    cfg.seed = seed;
    cfg.power = q;
    cfg.reorthonormalize = reorth != 0;
    auto id = randomized_id(from_ptr(m, n, a, lda), k, cfg);
    to_idx(id.pivots, pivots);
    to_ptr(id.coeff, coeff);
  });
}

// sketch.hpp:200-223 with power iterations
int lref_randomized_id_power(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int oversample, int q,
                             int reorth, uint64_t seed, int64_t* pivots, double* coeff) {
  return guard([&] {
    SketchConfig cfg;
    cfg.oversample = oversample;
    cfg.seed = seed;
    cfg.power = q;
    cfg.reorthonormalize = reorth != 0;
    auto id = randomized_id(from_ptr(m, n, a, lda), k, cfg);
    to_idx(id.pivots, pivots);
    to_ptr(id.coeff, coeff);
  });
}

// tsID from a column ID: row pivots, row coeff, skeleton
int lref_tsid_from_column_id(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                             const int64_t* col_pivots, const double* col_coeff, int64_t* row_pivots,
                             double* row_coeff, double* skeleton) {
  return guard([&] {
    ColumnId<double> cid;
    cid.cols = n;
    cid.rank = k;
    cid.pivots = from_idx(n, col_pivots);
    cid.coeff = from_ptr(k, n - k, col_coeff, k);
    auto ts = tsid_from_column_id(from_ptr(m, n, a, lda), cid);
    to_idx(ts.row_id.pivots, row_pivots);
    to_ptr(ts.row_id.coeff, row_coeff);
    to_ptr(ts.skeleton, skeleton);
  });
}

// CUR from stored pivots: u_mode 0 = cur.hpp:30, 1 = lowrank_main.cpp:215
int lref_cur_from_two_sided(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                            const int64_t* col_pivots, const double* col_coeff, const int64_t* row_pivots,
                            const double* row_coeff, double thr, int u_mode, double* c, double* u,
                            double* r) {
  return guard([&] {
    const Mat A = from_ptr(m, n, a, lda);
    TwoSidedId<double> ts;
    ts.col_id.cols = n;
    ts.col_id.rank = k;
    ts.col_id.pivots = from_idx(n, col_pivots);
    ts.col_id.coeff = from_ptr(k, n - k, col_coeff, k);
    ts.row_id.rows = m;
    ts.row_id.rank = k;
    ts.row_id.pivots = from_idx(m, row_pivots);
    ts.row_id.coeff = from_ptr(k, m - k, row_coeff, k);
    auto cur = cur_from_two_sided(A, ts, thr);
    if (u_mode == 1) cur.u = pinv(cur.c, thr) * A * pinv(cur.r, thr);
    to_ptr(cur.c, c);
    to_ptr(cur.u, u);
    to_ptr(cur.r, r);
  });
}

// Full pipelines (the CLI cur-id-rand and cur-pinv paths, lowrank_main.cpp:199-216)
int lref_randomized_cur(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, int oversample,
                        uint64_t seed, double thr, int u_mode, int64_t* col_pivots, int64_t* row_pivots,
                        double* c, double* u, double* r) {
  return guard([&] {
    const Mat A = from_ptr(m, n, a, lda);
    SketchConfig cfg;
    cfg.oversample = oversample;
    cfg.seed = seed;
    auto cur = randomized_cur(A, k, cfg, SolveStrategy::automatic(), thr);
    if (u_mode == 1) cur.u = pinv(cur.c, thr) * A * pinv(cur.r, thr);
    to_idx(cur.col_pivots, col_pivots);
    to_idx(cur.row_pivots, row_pivots);
    to_ptr(cur.c, c);
    to_ptr(cur.u, u);
    to_ptr(cur.r, r);
  });
}

int lref_cur_id(int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, double thr, int u_mode,
                int64_t* col_pivots, int64_t* row_pivots, double* c, double* u, double* r) {
  return guard([&] {
    const Mat A = from_ptr(m, n, a, lda);
    auto cur = cur_id(A, k, SolveStrategy::automatic(), thr);
    if (u_mode == 1) cur.u = pinv(cur.c, thr) * A * pinv(cur.r, thr);
    to_idx(cur.col_pivots, col_pivots);
    to_idx(cur.row_pivots, row_pivots);
    to_ptr(cur.c, c);
    to_ptr(cur.u, u);
    to_ptr(cur.r, r);
  });
}

}  // extern "C"
