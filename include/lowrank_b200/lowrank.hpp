// lowrank_b200/lowrank.hpp -- C++ drop-in for the reference library's hot
// path (namespace lowrank, /root/reference/proj/include/lowrank), running on
// the B200 through the C ABI of lowrank_b200.h.
//
// Same names, structs, defaults and exception types as the reference:
//   types / exceptions      core.hpp:12-42
//   gaussian_matrix         rng.hpp:74-94
//   cpqr_partial / _full    cpqr.hpp:32-122
//   SolveStrategy / stabilized_coeff_solve   solve.hpp:9-145
//   Svd / svd / pinv / spectral_norm         svd.hpp:16-207
//   ColumnId / RowId / TwoSidedId / id_*     id.hpp:12-159
//   CurDecomposition / cur_from_two_sided / cur_id / reconstruct  cur.hpp:9-80
//   SketchConfig / SampleMatrix / sketch_gaussian / sketch_srft /
//   srft_operator / sketch_power / randomized_id / randomized_cur /
//   randomized_svd          sketch.hpp:21-254; orth_rows svd.hpp:216-235
// Templates accept any Eigen::MatrixBase<Derived> with Scalar = double (the
// B200 path is FP64; other scalars fail at compile time -- there is no CPU
// fallback).  Needs <Eigen/Dense> (Eigen 3.4, or oracle/eigen_subset).
#pragma once

#include <Eigen/Dense>

#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../lowrank_b200.h"

namespace lowrank {

using Index = Eigen::Index;
template <typename Scalar>
using MatrixX = Eigen::Matrix<Scalar, Eigen::Dynamic, Eigen::Dynamic>;
template <typename Scalar>
using VectorX = Eigen::Matrix<Scalar, Eigen::Dynamic, 1>;
using IndexVector = Eigen::Matrix<Index, Eigen::Dynamic, 1>;

class SingularityError : public std::runtime_error {
 public:
  SingularityError(const std::string& what, Index index) : std::runtime_error(what), index_(index) {}
  Index index() const { return index_; }

 private:
  Index index_;
};
class ConvergenceError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class ParseError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
/// Device / driver failure (no CPU fallback exists).
class DeviceError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace b200 {

inline void check(int rc) {
  if (rc == LR_OK) return;
  const std::string msg = lr_last_error();
  switch (rc) {
    case LR_EINVAL: throw std::invalid_argument(msg);
    case LR_ESINGULAR: throw SingularityError(msg, static_cast<Index>(lr_last_singular_index()));
    case LR_ECONVERGE: throw ConvergenceError(msg);
    case LR_ECUDA: throw DeviceError(msg);
    case LR_EPARSE: throw ParseError(msg);
    default: throw std::runtime_error(msg);
  }
}

/// Process-wide context on device 0 (create your own lr_ctx for other devices).
inline lr_ctx* context() {
  static std::unique_ptr<lr_ctx, int (*)(lr_ctx*)> ctx = [] {
    lr_ctx* c = nullptr;
    check(lr_ctx_create(&c, 0));
    return std::unique_ptr<lr_ctx, int (*)(lr_ctx*)>(c, lr_ctx_destroy);
  }();
  return ctx.get();
}

template <typename Derived>
MatrixX<double> dense(const Eigen::MatrixBase<Derived>& a) {
  static_assert(std::is_same<typename Derived::Scalar, double>::value,
                "lowrank_b200: the B200 path is FP64 only");
  return MatrixX<double>(a);
}

inline IndexVector to_index(const std::vector<int64_t>& v) {
  IndexVector out(static_cast<Index>(v.size()));
  for (size_t i = 0; i < v.size(); ++i) out(static_cast<Index>(i)) = v[i];
  return out;
}
inline std::vector<int64_t> from_index(const IndexVector& p) {
  std::vector<int64_t> out(static_cast<size_t>(p.size()));
  for (Index i = 0; i < p.size(); ++i) out[static_cast<size_t>(i)] = p(i);
  return out;
}
inline Index ld(const MatrixX<double>& a) { return std::max<Index>(1, a.rows()); }

/// a * b on the GPU (lr_gemm): the reconstruction products stay off the host
inline MatrixX<double> matmul(const MatrixX<double>& a, const MatrixX<double>& b) {
  if (a.cols() != b.rows()) throw std::invalid_argument("matmul: inner dimensions differ");
  MatrixX<double> c(a.rows(), b.cols());
  if (c.rows() == 0 || c.cols() == 0) return c;
  if (a.cols() == 0) {
    c.setZero();
    return c;
  }
  check(lr_gemm(context(), a.rows(), b.cols(), a.cols(), a.data(), ld(a), b.data(), ld(b), c.data(), ld(c)));
  return c;
}

}  // namespace b200

// ---------------------------------------------------------------- core.hpp
template <typename Derived>
void require_nonempty(const Eigen::MatrixBase<Derived>& a, const char* who) {
  if (a.rows() < 1 || a.cols() < 1) throw std::invalid_argument(std::string(who) + ": matrix must be nonempty");
}
template <typename Derived>
void require_finite(const Eigen::MatrixBase<Derived>& a, const char* who) {
  if (!a.allFinite()) throw std::invalid_argument(std::string(who) + ": matrix has non-finite entries");
}
inline void require_rank_in_range(Index k, Index rows, Index cols, const char* who) {
  if (k < 1 || k > std::min(rows, cols))
    throw std::invalid_argument(std::string(who) + ": rank " + std::to_string(k) + " out of range for " +
                                std::to_string(rows) + "x" + std::to_string(cols) + " matrix");
}
template <typename Derived>
typename Derived::Scalar frobenius_norm(const Eigen::MatrixBase<Derived>& a) {
  return a.norm();
}
template <typename Derived>
MatrixX<typename Derived::Scalar> select_columns(const Eigen::MatrixBase<Derived>& a, const IndexVector& pivots,
                                                 Index count) {
  MatrixX<typename Derived::Scalar> out(a.rows(), count);
  for (Index j = 0; j < count; ++j) out.col(j) = a.col(pivots(j));
  return out;
}
template <typename Derived>
MatrixX<typename Derived::Scalar> select_rows(const Eigen::MatrixBase<Derived>& a, const IndexVector& pivots,
                                              Index count) {
  MatrixX<typename Derived::Scalar> out(count, a.cols());
  for (Index i = 0; i < count; ++i) out.row(i) = a.row(pivots(i));
  return out;
}

// ---------------------------------------------------------------- rng.hpp
namespace detail {
inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
}  // namespace detail

/// rng.hpp:27-29 (counter-mode SplitMix64; integer-exact host helper)
inline std::uint64_t stream_value(std::uint64_t seed, std::uint64_t index) {
  return detail::mix64(seed + (index + 1) * 0x9E3779B97F4A7C15ULL);
}
/// rng.hpp:32-34
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) {
  return stream_value(seed, tag ^ 0xD1B54A32D192ED03ULL);
}

/// rng.hpp:37-67 (sequential view over one stream; host-side, test-matrix generation)
class CounterRng {
 public:
  explicit CounterRng(std::uint64_t seed) : seed_(seed) {}
  std::uint64_t next_u64() { return stream_value(seed_, next_++); }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  Index next_index(Index bound) { return static_cast<Index>(next_u64() % static_cast<std::uint64_t>(bound)); }
  std::vector<Index> sample_without_replacement(Index population, Index count) {
    std::vector<Index> pool(static_cast<std::size_t>(population));
    for (Index i = 0; i < population; ++i) pool[static_cast<std::size_t>(i)] = i;
    for (Index i = 0; i < count; ++i) {
      Index j = i + next_index(population - i);
      std::swap(pool[static_cast<std::size_t>(i)], pool[static_cast<std::size_t>(j)]);
    }
    pool.resize(static_cast<std::size_t>(count));
    return pool;
  }

 private:
  std::uint64_t seed_;
  std::uint64_t next_ = 0;
};

/// rng.hpp:74-94, generated on the GPU
template <typename Scalar = double>
MatrixX<Scalar> gaussian_matrix(Index rows, Index cols, std::uint64_t seed) {
  static_assert(std::is_same<Scalar, double>::value, "lowrank_b200: the B200 path is FP64 only");
  if (rows < 1 || cols < 1) throw std::invalid_argument("gaussian_matrix: dimensions must be positive");
  MatrixX<double> out(rows, cols);
  b200::check(lr_gaussian_matrix(b200::context(), rows, cols, seed, out.data()));
  return out;
}

// ---------------------------------------------------------------- cpqr.hpp
template <typename Scalar>
struct PivotedQr {
  MatrixX<Scalar> q;
  MatrixX<Scalar> s;
  IndexVector pivots;
  Index rank_achieved = 0;
};

template <typename Derived>
PivotedQr<typename Derived::Scalar> cpqr_partial(const Eigen::MatrixBase<Derived>& a, Index k) {
  MatrixX<double> d = b200::dense(a);
  PivotedQr<double> out;
  const Index m = d.rows(), n = d.cols();
  const Index kk = std::max<Index>(k, 0);
  out.q.resize(m, kk);
  out.s.resize(kk, n);
  std::vector<int64_t> piv(static_cast<size_t>(std::max<Index>(n, 0)));
  b200::check(lr_cpqr_partial(b200::context(), m, n, d.data(), b200::ld(d), k, out.q.data(), out.s.data(),
                              piv.data()));
  out.pivots = b200::to_index(piv);
  out.rank_achieved = k;
  return out;
}

template <typename Derived>
PivotedQr<typename Derived::Scalar> cpqr_full(const Eigen::MatrixBase<Derived>& a) {
  require_nonempty(a, "cpqr_full");
  return cpqr_partial(a, std::min(a.rows(), a.cols()));
}

// ---------------------------------------------------------------- solve.hpp
enum class SolveKind { BackSubstitution, TruncatedPinv, Tikhonov };

struct SolveStrategy {
  SolveKind kind = SolveKind::BackSubstitution;
  double threshold = 1e-12;
  double ridge = 0.0;
  bool escalate = true;

  static SolveStrategy automatic() { return {}; }
  static SolveStrategy back_substitution(double threshold = 1e-12) {
    return {SolveKind::BackSubstitution, threshold, 0.0, false};
  }
  static SolveStrategy truncated_pinv(double threshold = 1e-12) {
    return {SolveKind::TruncatedPinv, threshold, 0.0, false};
  }
  static SolveStrategy tikhonov(double ridge, double threshold = 1e-12) {
    return {SolveKind::Tikhonov, threshold, ridge, false};
  }
  lr_solve_strategy c_abi() const {
    return {static_cast<int>(kind), threshold, ridge, escalate ? 1 : 0};
  }
};

template <typename Scalar>
MatrixX<Scalar> stabilized_coeff_solve(const MatrixX<Scalar>& s11, const MatrixX<Scalar>& s12,
                                       const SolveStrategy& strategy = SolveStrategy::automatic()) {
  static_assert(std::is_same<Scalar, double>::value, "lowrank_b200: the B200 path is FP64 only");
  if (s11.rows() != s11.cols()) throw std::invalid_argument("stabilized_coeff_solve: triangular block must be square");
  if (s12.rows() != s11.rows()) throw std::invalid_argument("stabilized_coeff_solve: row count mismatch");
  MatrixX<double> t(s11.rows(), s12.cols());
  if (s11.rows() == 0) return t;
  b200::check(lr_stabilized_coeff_solve(b200::context(), s11.rows(), s12.cols(), s11.data(), b200::ld(s11),
                                        s12.data(), b200::ld(s12), strategy.c_abi(), t.data()));
  return t;
}

// ---------------------------------------------------------------- svd.hpp
template <typename Scalar>
struct Svd {
  MatrixX<Scalar> u;
  VectorX<Scalar> sigma;
  MatrixX<Scalar> v;

  Index rank(Scalar rel_threshold) const {
    if (sigma.size() == 0 || sigma(0) == Scalar(0)) return 0;
    Index r = 0;
    while (r < sigma.size() && sigma(r) >= rel_threshold * sigma(0)) ++r;
    return r;
  }
};

template <typename Derived>
Svd<typename Derived::Scalar> svd(const Eigen::MatrixBase<Derived>& a) {
  MatrixX<double> d = b200::dense(a);
  const Index m = d.rows(), n = d.cols(), r = std::min(m, n);
  Svd<double> out;
  out.u.resize(m, r);
  out.sigma.resize(r);
  out.v.resize(n, r);
  b200::check(lr_svd(b200::context(), m, n, d.data(), b200::ld(d), out.u.data(), out.sigma.data(), out.v.data()));
  return out;
}

template <typename Derived>
typename Derived::Scalar spectral_norm(const Eigen::MatrixBase<Derived>& a) {
  return svd(a).sigma(0);
}

template <typename Derived>
MatrixX<typename Derived::Scalar> pinv(const Eigen::MatrixBase<Derived>& a, double threshold = 1e-12) {
  MatrixX<double> d = b200::dense(a);
  MatrixX<double> out(d.cols(), d.rows());
  b200::check(lr_pinv(b200::context(), d.rows(), d.cols(), d.data(), b200::ld(d), threshold, out.data()));
  return out;
}

// ---------------------------------------------------------------- id.hpp
template <typename Scalar>
struct ColumnId {
  Index cols = 0;
  Index rank = 0;
  IndexVector pivots;
  MatrixX<Scalar> coeff;

  MatrixX<Scalar> basis() const {
    MatrixX<Scalar> v = MatrixX<Scalar>::Zero(cols, rank);
    for (Index l = 0; l < cols; ++l) {
      if (l < rank)
        v(pivots(l), l) = Scalar(1);
      else
        v.row(pivots(l)) = coeff.col(l - rank).transpose();
    }
    return v;
  }
};

template <typename Scalar>
struct RowId {
  Index rows = 0;
  Index rank = 0;
  IndexVector pivots;
  MatrixX<Scalar> coeff;

  MatrixX<Scalar> basis() const {
    MatrixX<Scalar> w = MatrixX<Scalar>::Zero(rows, rank);
    for (Index l = 0; l < rows; ++l) {
      if (l < rank)
        w(pivots(l), l) = Scalar(1);
      else
        w.row(pivots(l)) = coeff.col(l - rank).transpose();
    }
    return w;
  }
};

template <typename Scalar>
struct TwoSidedId {
  ColumnId<Scalar> col_id;
  RowId<Scalar> row_id;
  MatrixX<Scalar> skeleton;

  const IndexVector& col_pivots() const { return col_id.pivots; }
  const IndexVector& row_pivots() const { return row_id.pivots; }
  MatrixX<Scalar> col_basis() const { return col_id.basis(); }
  MatrixX<Scalar> row_basis() const { return row_id.basis(); }
  Index rank() const { return col_id.rank; }
};

template <typename Derived, typename Scalar = typename Derived::Scalar>
MatrixX<Scalar> skeleton_columns(const Eigen::MatrixBase<Derived>& a, const ColumnId<Scalar>& id) {
  return select_columns(a, id.pivots, id.rank);
}
template <typename Derived, typename Scalar = typename Derived::Scalar>
MatrixX<Scalar> skeleton_rows(const Eigen::MatrixBase<Derived>& a, const RowId<Scalar>& id) {
  return select_rows(a, id.pivots, id.rank);
}

template <typename Derived>
ColumnId<typename Derived::Scalar> id_column(const Eigen::MatrixBase<Derived>& a, Index k,
                                             const SolveStrategy& strategy = SolveStrategy::automatic()) {
  MatrixX<double> d = b200::dense(a);
  const Index m = d.rows(), n = d.cols();
  ColumnId<double> id;
  id.cols = n;
  id.rank = k;
  std::vector<int64_t> piv(static_cast<size_t>(std::max<Index>(n, 0)));
  id.coeff.resize(std::max<Index>(k, 0), std::max<Index>(n - std::max<Index>(k, 0), 0));
  b200::check(lr_id_column(b200::context(), m, n, d.data(), b200::ld(d), k, strategy.c_abi(), piv.data(),
                           id.coeff.data()));
  id.pivots = b200::to_index(piv);
  return id;
}

template <typename Derived>
RowId<typename Derived::Scalar> id_row(const Eigen::MatrixBase<Derived>& a, Index k,
                                       const SolveStrategy& strategy = SolveStrategy::automatic()) {
  MatrixX<double> d = b200::dense(a);
  const Index m = d.rows(), n = d.cols();
  RowId<double> id;
  id.rows = m;
  id.rank = k;
  std::vector<int64_t> piv(static_cast<size_t>(std::max<Index>(m, 0)));
  id.coeff.resize(std::max<Index>(k, 0), std::max<Index>(m - std::max<Index>(k, 0), 0));
  b200::check(lr_id_row(b200::context(), m, n, d.data(), b200::ld(d), k, strategy.c_abi(), piv.data(),
                        id.coeff.data()));
  id.pivots = b200::to_index(piv);
  return id;
}

template <typename Derived, typename Scalar = typename Derived::Scalar>
TwoSidedId<Scalar> tsid_from_column_id(const Eigen::MatrixBase<Derived>& a, ColumnId<Scalar> col_id,
                                       const SolveStrategy& strategy = SolveStrategy::automatic()) {
  MatrixX<double> d = b200::dense(a);
  const Index m = d.rows(), n = d.cols(), k = col_id.rank;
  TwoSidedId<double> out;
  std::vector<int64_t> cp = b200::from_index(col_id.pivots), rp(static_cast<size_t>(m));
  out.row_id.rows = m;
  out.row_id.rank = k;
  out.row_id.coeff.resize(k, std::max<Index>(m - k, 0));
  out.skeleton.resize(k, k);
  b200::check(lr_tsid_from_column_id(b200::context(), m, n, d.data(), b200::ld(d), k, cp.data(), strategy.c_abi(),
                                     rp.data(), out.row_id.coeff.data(), out.skeleton.data()));
  out.row_id.pivots = b200::to_index(rp);
  out.col_id = std::move(col_id);
  return out;
}

template <typename Derived>
TwoSidedId<typename Derived::Scalar> id_two_sided(const Eigen::MatrixBase<Derived>& a, Index k,
                                                  const SolveStrategy& strategy = SolveStrategy::automatic()) {
  return tsid_from_column_id(a, id_column(a, k, strategy), strategy);
}

template <typename Derived, typename Scalar = typename Derived::Scalar>
MatrixX<Scalar> reconstruct(const Eigen::MatrixBase<Derived>& a, const ColumnId<Scalar>& id) {
  return b200::matmul(skeleton_columns(a, id), MatrixX<Scalar>(id.basis().transpose()));
}
template <typename Derived, typename Scalar = typename Derived::Scalar>
MatrixX<Scalar> reconstruct(const Eigen::MatrixBase<Derived>& a, const RowId<Scalar>& id) {
  return b200::matmul(id.basis(), skeleton_rows(a, id));
}
template <typename Scalar>
MatrixX<Scalar> reconstruct(const TwoSidedId<Scalar>& tsid) {
  return b200::matmul(b200::matmul(tsid.row_basis(), tsid.skeleton), MatrixX<Scalar>(tsid.col_basis().transpose()));
}

// ---------------------------------------------------------------- cur.hpp
template <typename Scalar>
struct CurDecomposition {
  MatrixX<Scalar> c;
  MatrixX<Scalar> u;
  MatrixX<Scalar> r;
  IndexVector col_pivots;
  IndexVector row_pivots;

  Index rank() const { return u.rows(); }
};

/// cur.hpp:23-34 (u_mode LR_U_VT_RPINV); LR_U_CPINV_A_RPINV gives the
/// lowrank_main.cpp:215 middle factor pinv(c) a pinv(r).
template <typename Derived, typename Scalar = typename Derived::Scalar>
CurDecomposition<Scalar> cur_from_two_sided(const Eigen::MatrixBase<Derived>& a, const TwoSidedId<Scalar>& tsid,
                                            double pinv_threshold = 1e-12, int u_mode = LR_U_VT_RPINV) {
  MatrixX<double> d = b200::dense(a);
  const Index m = d.rows(), n = d.cols(), k = tsid.rank();
  CurDecomposition<double> cur;
  cur.c.resize(m, k);
  cur.u.resize(k, k);
  cur.r.resize(k, n);
  std::vector<int64_t> cp = b200::from_index(tsid.col_pivots()), rp = b200::from_index(tsid.row_pivots());
  MatrixX<double> cc = tsid.col_id.coeff;
  b200::check(lr_cur_from_two_sided(b200::context(), m, n, d.data(), b200::ld(d), k, cp.data(),
                                    cc.size() ? cc.data() : nullptr, rp.data(), pinv_threshold, u_mode, cur.c.data(),
                                    cur.u.data(), cur.r.data()));
  cur.col_pivots = tsid.col_pivots();
  cur.row_pivots = tsid.row_pivots();
  return cur;
}

template <typename Derived>
CurDecomposition<typename Derived::Scalar> cur_id(const Eigen::MatrixBase<Derived>& a, Index k,
                                                  const SolveStrategy& strategy = SolveStrategy::automatic(),
                                                  double pinv_threshold = 1e-12) {
  return cur_from_two_sided(a, id_two_sided(a, k, strategy), pinv_threshold);
}

template <typename Scalar>
MatrixX<Scalar> reconstruct(const CurDecomposition<Scalar>& cur) {
  return b200::matmul(b200::matmul(cur.c, cur.u), cur.r);
}

/// cur.hpp:52-74 (Eq. 31 variant; not on the hot path): the same
/// composition as the reference, with both pseudoinverses on the GPU.
template <typename Derived, typename Scalar = typename Derived::Scalar>
MatrixX<Scalar> cur_refined_u(const Eigen::MatrixBase<Derived>& a, const CurDecomposition<Scalar>& cur,
                              const ColumnId<Scalar>& col_id, const PivotedQr<Scalar>& qr,
                              double pinv_threshold = 1e-12) {
  const Index k = cur.rank();
  if (col_id.rank != k || qr.rank_achieved != k) throw std::invalid_argument("cur_refined_u: factor ranks disagree");
  if (col_id.cols != a.cols() || qr.pivots.size() != a.cols() || cur.c.rows() != a.rows() || cur.r.cols() != a.cols())
    throw std::invalid_argument("cur_refined_u: factor shapes disagree");
  for (Index j = 0; j < a.cols(); ++j)
    if (col_id.pivots(j) != qr.pivots(j)) throw std::invalid_argument("cur_refined_u: pivot sequences disagree");
  MatrixX<Scalar> residual = a;
  const MatrixX<Scalar> qs = b200::matmul(qr.q, qr.s);
  for (Index j = 0; j < a.cols(); ++j) residual.col(qr.pivots(j)) -= qs.col(j);
  const MatrixX<Scalar> rhs =
      MatrixX<Scalar>(col_id.basis().transpose()) + b200::matmul(pinv(cur.c, pinv_threshold), residual);
  return b200::matmul(rhs, pinv(cur.r, pinv_threshold));
}

// ---------------------------------------------------------------- sketch.hpp
enum class SketchKind { Gaussian, Srft };

struct SketchConfig {
  SketchKind kind = SketchKind::Gaussian;
  int oversample = 10;
  Index srft_samples = 0;
  int power = 0;
  bool reorthonormalize = true;
  std::uint64_t seed = 0;

  Index sample_count(Index k) const {
    if (kind == SketchKind::Gaussian) return k + static_cast<Index>(oversample);
    return srft_samples > 0 ? srft_samples : 2 * k;
  }
  lr_sketch_config c_abi() const {
    return {static_cast<int>(kind), oversample, static_cast<int64_t>(srft_samples), power, reorthonormalize ? 1 : 0,
            seed};
  }
};

struct SampleProvenance {
  SketchKind kind = SketchKind::Gaussian;
  Index samples = 0;
  int power = 0;
  bool reorthonormalized = false;
  std::uint64_t seed = 0;
};

template <typename Scalar>
struct SampleMatrix {
  MatrixX<Scalar> y;
  SampleProvenance provenance;
};

template <typename Derived>
SampleMatrix<typename Derived::Scalar> sketch_gaussian(const Eigen::MatrixBase<Derived>& a, Index ell,
                                                       std::uint64_t seed) {
  MatrixX<double> d = b200::dense(a);
  SampleMatrix<double> out;
  out.y.resize(std::max<Index>(ell, 0), d.cols());
  b200::check(lr_sketch_gaussian(b200::context(), d.rows(), d.cols(), d.data(), b200::ld(d), ell, seed,
                                 out.y.data()));
  out.provenance = {SketchKind::Gaussian, ell, 0, false, seed};
  return out;
}

// sketch.hpp:84-100
template <typename Scalar = double>
MatrixX<Scalar> srft_operator(Index m, Index ell, std::uint64_t seed) {
  static_assert(std::is_same_v<Scalar, double>, "the B200 path is FP64 only");
  MatrixX<double> out(std::max<Index>(ell, 0), std::max<Index>(m, 0));
  b200::check(lr_srft_operator(b200::context(), m, ell, seed, out.data()));
  return out;
}

// sketch.hpp:110-143
template <typename Derived>
SampleMatrix<typename Derived::Scalar> sketch_srft(const Eigen::MatrixBase<Derived>& a, Index ell,
                                                   std::uint64_t seed) {
  MatrixX<double> d = b200::dense(a);
  SampleMatrix<double> out;
  out.y.resize(std::max<Index>(ell, 0), d.cols());
  b200::check(lr_sketch_srft(b200::context(), d.rows(), d.cols(), d.data(), b200::ld(d), ell, seed, out.y.data()));
  out.provenance = {SketchKind::Srft, ell, 0, false, seed};
  return out;
}

// svd.hpp:216-235
template <typename Derived>
MatrixX<typename Derived::Scalar> orth_rows(const Eigen::MatrixBase<Derived>& y) {
  MatrixX<double> d = b200::dense(y);
  MatrixX<double> out(d.rows(), d.cols());
  int64_t r = 0;
  b200::check(lr_orth_rows(b200::context(), d.rows(), d.cols(), d.data(), b200::ld(d), out.data(), &r));
  return MatrixX<double>(out.topRows(r));
}

// sketch.hpp:148-164
template <typename Derived>
SampleMatrix<typename Derived::Scalar> sketch_power(const Eigen::MatrixBase<Derived>& a, Index ell, int q,
                                                    bool reorthonormalize, std::uint64_t seed) {
  MatrixX<double> d = b200::dense(a);
  MatrixX<double> y(std::max<Index>(ell, 0), d.cols());
  int64_t rows = 0;
  b200::check(lr_sketch_power(b200::context(), d.rows(), d.cols(), d.data(), b200::ld(d), ell, q,
                              reorthonormalize ? 1 : 0, seed, y.data(), &rows));
  SampleMatrix<double> out;
  out.y = y.topRows(rows);
  out.provenance = {SketchKind::Gaussian, ell, q, reorthonormalize && q > 0, seed};
  return out;
}

// sketch.hpp:238-254
template <typename Derived>
Svd<typename Derived::Scalar> randomized_svd(const Eigen::MatrixBase<Derived>& a, Index k, const SketchConfig& cfg) {
  MatrixX<double> d = b200::dense(a);
  const Index m = d.rows(), n = d.cols(), kk = std::max<Index>(k, 0);
  Svd<double> out;
  out.u.resize(m, kk);
  out.sigma.resize(kk);
  out.v.resize(n, kk);
  b200::check(lr_randomized_svd(b200::context(), m, n, d.data(), b200::ld(d), k, cfg.c_abi(), out.u.data(),
                                out.sigma.data(), out.v.data()));
  return out;
}

template <typename Derived>
ColumnId<typename Derived::Scalar> randomized_id(const Eigen::MatrixBase<Derived>& a, Index k,
                                                 const SketchConfig& cfg,
                                                 const SolveStrategy& strategy = SolveStrategy::automatic()) {
  MatrixX<double> d = b200::dense(a);
  const Index m = d.rows(), n = d.cols();
  ColumnId<double> id;
  id.cols = n;
  id.rank = k;
  std::vector<int64_t> piv(static_cast<size_t>(std::max<Index>(n, 0)));
  id.coeff.resize(std::max<Index>(k, 0), std::max<Index>(n - std::max<Index>(k, 0), 0));
  b200::check(lr_randomized_id(b200::context(), m, n, d.data(), b200::ld(d), k, cfg.c_abi(), strategy.c_abi(),
                               piv.data(), id.coeff.data()));
  id.pivots = b200::to_index(piv);
  return id;
}

template <typename Derived>
CurDecomposition<typename Derived::Scalar> randomized_cur(const Eigen::MatrixBase<Derived>& a, Index k,
                                                          const SketchConfig& cfg,
                                                          const SolveStrategy& strategy = SolveStrategy::automatic(),
                                                          double pinv_threshold = 1e-12,
                                                          int u_mode = LR_U_VT_RPINV) {
  MatrixX<double> d = b200::dense(a);
  const Index m = d.rows(), n = d.cols();
  require_rank_in_range(k, m, n, "randomized_id");
  CurDecomposition<double> cur;
  cur.c.resize(m, k);
  cur.u.resize(k, k);
  cur.r.resize(k, n);
  std::vector<int64_t> cp(static_cast<size_t>(n)), rp(static_cast<size_t>(m));
  b200::check(lr_randomized_cur(b200::context(), m, n, d.data(), b200::ld(d), k, cfg.c_abi(), strategy.c_abi(),
                                pinv_threshold, u_mode, cp.data(), rp.data(), cur.c.data(), cur.u.data(),
                                cur.r.data(), nullptr, nullptr, nullptr));
  cur.col_pivots = b200::to_index(cp);
  cur.row_pivots = b200::to_index(rp);
  return cur;
}

}  // namespace lowrank
