"""Edge cases of the coefficient solve and of the pseudoinverse on the GPU
against the CPU oracle (solve.hpp:37-145, svd.hpp:193-207).

* pinv / CUR with a LOOSE threshold (1e-3) on tall and wide matrices whose
  condition number (1e4) puts singular values below the cutoff: the
  CholeskyQR2 fast path must not run (it would return the untruncated
  inverse), the truncated SVD route must (svd.hpp:201-205);
* Tikhonov with ridge = 0 on a singular S11: the normal matrix is singular,
  the Cholesky breaks down and the reference's conjugate gradients give the
  answer (solve.hpp:37-57, :133-142);
* back-substitution on CPQR-produced S11 whose diagonal ratio is 1e8-1e9,
  just below the 1e10 escalation limit (solve.hpp:62-89, :119-126): the GPU
  applies an explicit back-substitution operator, the reference solves row
  by row; both must agree to 1e-10.
"""
import numpy as np
import pytest

from oracle_lib import rel
from paper_1412_8447_b200 import inputs

pytestmark = pytest.mark.gpu
TOL = 1e-10


def graded(rows, cols, smax, smin, seed):
    """U diag(s) V^T with log-spaced singular values smax .. smin."""
    r = min(rows, cols)
    u = inputs.haar_np(rows, r, seed)
    v = inputs.haar_np(cols, r, seed + 1)
    s = np.logspace(np.log10(smax), np.log10(smin), r)
    return np.asfortranarray((u * s) @ v.T), s


@pytest.mark.parametrize("shape", [(400, 40), (40, 400), (1000, 64)])
def test_pinv_loose_threshold_truncates(lr, oracle, shape):
    a, s = graded(*shape, 1.0, 1e-4, 31)
    thr = 1e-3
    p = lr.pinv(a, thr)
    po = oracle.pinv(a, thr)
    assert rel(p, po) <= TOL
    assert lr.default_context().stats()["pinv_fast_path"] == 0
    # the truncated pinv has norm 1/min{s_i >= thr s_1}, far below 1/s_min
    assert np.linalg.norm(p, 2) == pytest.approx(1.0 / s[s >= thr * s[0]].min(), rel=1e-8)
    # a threshold below 1/cond keeps every singular value: the fast path is allowed
    p2 = lr.pinv(a, 1e-12)
    assert rel(p2, oracle.pinv(a, 1e-12)) <= 1e-9


@pytest.mark.parametrize("mode", [0, 1])
def test_cur_loose_pinv_threshold(lr, oracle, mode):
    # rank-64 matrix with a 1e4 spread, CUR of rank 48: C and R keep the spread
    u = inputs.haar_np(600, 64, 41)
    v = inputs.haar_np(500, 64, 42)
    a = np.asfortranarray((u * np.logspace(0, -4, 64)) @ v.T)
    k, thr = 48, 1e-3
    cur = lr.cur_id(a, k, pinv_threshold=thr, u_mode=mode)
    o = oracle.cur_id(a, k, u_mode=mode, thr=thr)
    assert np.array_equal(cur.col_pivots, o["col_pivots"]) and np.array_equal(cur.row_pivots, o["row_pivots"])
    assert rel(cur.u, o["u"]) <= 1e-9


def test_tikhonov_ridge_zero_singular(lr, oracle):
    s11 = np.triu(oracle.gaussian_matrix(30, 30, 23) + 6.0 * np.eye(30))
    s11[:, 11] = 0.0  # exactly singular: a zero column (normal matrix row/column 11 = 0)
    s12 = oracle.gaussian_matrix(30, 257, 24)
    strat = lr.SolveStrategy(2, 1e-12, 0.0, False)
    t = lr.stabilized_coeff_solve(s11, s12, strat)
    to = oracle.coeff_solve(s11, s12, 2, 1e-12, 0.0, 0)
    assert np.all(np.isfinite(t))
    assert rel(t, to) <= 1e-9
    assert np.all(t[11] == 0.0)


def test_tikhonov_ridge_positive_matches(lr, oracle):
    s11 = np.triu(oracle.gaussian_matrix(50, 50, 3) + 4.0 * np.eye(50))
    s12 = oracle.gaussian_matrix(50, 123, 4)
    strat = lr.SolveStrategy(2, 1e-12, 0.05, False)
    assert rel(lr.stabilized_coeff_solve(s11, s12, strat), oracle.coeff_solve(s11, s12, 2, 1e-12, 0.05, 0)) <= TOL


def graded_k(rows, cols, k, smin, seed):
    """Spectrum log-spaced 1 .. smin over the first k values, smin 1e-3 beyond:
    the CPQR's leading k x k block then has a diagonal ratio of ~1/smin."""
    r = min(rows, cols)
    u = inputs.haar_np(rows, r, seed)
    v = inputs.haar_np(cols, r, seed + 1)
    s = np.concatenate([np.logspace(0, np.log10(smin), k), np.full(r - k, smin * 1e-3)])
    return np.asfortranarray((u * s) @ v.T)


@pytest.mark.parametrize("smin,k", [(1e-8, 60), (1e-9, 60), (1e-10, 60), (5e-10, 100)])
def test_backsub_near_escalation_limit(lr, oracle, smin, k):
    a = graded_k(300, 400, k, smin, 57)
    q = oracle.cpqr(a, k, want_q=False)
    s11 = np.asfortranarray(q["s"][:, :k])
    s12 = np.asfortranarray(q["s"][:, k:])
    d = np.abs(np.diag(s11))
    assert 1e7 < d.max() / d.min() < 1e10  # below the escalation limit: back-substitution
    ctx = lr.default_context()
    ctx.reset_stats()
    t = lr.stabilized_coeff_solve(s11, s12)
    assert ctx.stats()["solve_escalated"] == 0
    assert rel(t, oracle.coeff_solve(s11, s12)) <= TOL
