"""GPU parity: the B200 path (through the C ABI) against the CPU oracle and the
golden fixtures produced by the reference's own code.

Tolerances (north_star): identical index sets; C, R, skeleton bit-exact;
ID/CUR factors and the relative Frobenius error within 1e-10 relative.
Gaussian entries: the integer stream is exact, CUDA's log/sincos give a
few-ulp difference from glibc (hard part 4).
"""
import os

import numpy as np
import pytest

from oracle_lib import rel
from paper_1412_8447_b200 import inputs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_small.npz")
TOL = 1e-10


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def ulp_close(a, b, ulps=8):
    scale = np.maximum(np.abs(a), np.abs(b))
    return np.all(np.abs(a - b) <= ulps * np.spacing(np.maximum(scale, 1e-300)))


# ------------------------------------------------------------------ rng / sketch
def test_gaussian_matrix_stream(lr, oracle):
    for rows, cols, seed in [(7, 5, 123), (5, 12, 3), (1, 1, 0), (33, 17, 2**63 + 11)]:
        g = lr.gaussian_matrix(rows, cols, seed)
        o = oracle.gaussian_matrix(rows, cols, seed)
        assert ulp_close(g, o, 8)
        assert np.array_equal(g, lr.gaussian_matrix(rows, cols, seed))


def test_sketch_of_identity_is_the_operator(lr):  # test_sketch.cpp:27-31
    y = lr.sketch_gaussian(np.eye(12), 5, 3).y
    assert np.array_equal(y, lr.gaussian_matrix(5, 12, 3))


def test_sketch_of_zero_is_zero(lr):  # test_sketch.cpp:33-36
    assert np.all(lr.sketch_gaussian(np.zeros((10, 6)), 4, 1).y == 0.0)


@pytest.mark.parametrize("shape,ell", [((300, 200), 37), ((1000, 129), 130), ((257, 1031), 64)])
def test_sketch_matches_oracle(lr, oracle, shape, ell):
    a = oracle.gaussian_matrix(*shape, 5)
    y = lr.sketch_gaussian(a, ell, 9).y
    assert rel(y, oracle.sketch_gaussian(a, ell, 9)) <= 1e-13


def test_sketch_validation(lr):  # test_sketch.cpp:50-54
    a = np.ones((6, 9))
    with pytest.raises(ValueError):
        lr.sketch_gaussian(a, 7, 1)
    bad = a.copy()
    bad[1, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        lr.sketch_gaussian(bad, 3, 1)


def test_gemm_kernel_vs_numpy(lr):
    import torch
    for (M, N, K) in [(510, 1000, 777), (128, 128, 16), (5, 7, 3), (300, 260, 4100)]:
        P = torch.randn(K, M, dtype=torch.float64, device="cuda")
        Q = torch.randn(K, N, dtype=torch.float64, device="cuda")
        Pc = lr.empty_colmajor(K, M, "cuda"); Pc.copy_(P)
        Qc = lr.empty_colmajor(K, N, "cuda"); Qc.copy_(Q)
        out = lr.empty_colmajor(M, N, "cuda")
        ctx = lr.default_context()
        torch.cuda.synchronize()  # inputs copied on torch's stream
        rc = ctx.lib.lr_gemm_tn_d(ctx.h, M, N, K, Pc.data_ptr(), Pc.stride(1), Qc.data_ptr(), Qc.stride(1),
                                  out.data_ptr(), out.stride(1))
        assert rc == 0, ctx.lib.lr_last_error()
        ctx.synchronize()
        ref = (P.T @ Q).cpu().numpy()
        assert rel(out.cpu().numpy(), ref) <= 1e-14


# ------------------------------------------------------------------ CPQR
def test_cpqr_golden(lr, gold):
    q = lr.cpqr_partial(gold["cpqr_a"], int(gold["cpqr_k"]))
    assert np.array_equal(q.pivots, gold["cpqr_piv"])
    assert rel(q.s, gold["cpqr_s"]) <= 1e-12 and rel(q.q, gold["cpqr_q"]) <= 1e-12
    f = lr.cpqr_full(gold["cpqrf_a"])
    assert np.array_equal(f.pivots, gold["cpqrf_piv"])
    assert rel(f.s, gold["cpqrf_s"]) <= 1e-12 and rel(f.q, gold["cpqrf_q"]) <= 1e-12


def test_cpqr_known_answers(lr):
    q = lr.cpqr_partial(np.eye(3), 2)  # test_cpqr.cpp:29-38
    assert list(q.pivots) == [0, 1, 2] and np.array_equal(q.s, [[1, 0, 0], [0, 1, 0]])
    a = np.zeros((2, 2)); a[0, 0], a[1, 1] = 1.0, 2.0  # :40-49
    q = lr.cpqr_partial(a, 2)
    assert list(q.pivots) == [1, 0] and abs(q.s[0, 0]) == pytest.approx(2.0)
    q = lr.cpqr_full(np.array([[5.0]]))  # :64-71
    assert q.q[0, 0] == pytest.approx(1.0) and q.s[0, 0] == pytest.approx(5.0)
    a = np.zeros((3, 4)); a[0, 1] = a[1, 2] = a[2, 3] = 2.0; a[0, 0] = 1.0  # ties -> lowest position
    assert list(lr.cpqr_partial(a, 3).pivots[:3]) == [1, 2, 3]


def test_cpqr_rank_deficient_and_det(lr, oracle):
    g = oracle.gaussian_matrix(6, 3, 11)
    dup = np.column_stack([g[:, 0], g[:, 1], g[:, 0], g[:, 2]])
    q = lr.cpqr_full(dup)
    assert abs(q.s[3, 3]) <= 1e-12 * abs(q.s[0, 0])
    assert np.linalg.norm(dup[:, q.pivots] - q.q @ q.s) <= 1e-12 * np.linalg.norm(dup)
    a = oracle.gaussian_matrix(12, 12, 3)
    q = lr.cpqr_full(a)
    assert np.prod(np.abs(np.diag(q.s))) == pytest.approx(abs(np.linalg.det(a)), rel=1e-8)


@pytest.mark.parametrize("shape,k", [((510, 3000), 510), ((500, 4096), 500), ((300, 5000), 300), ((310, 2000), 137),
                                     ((210, 6000), 210), ((256, 1500), 256), ((1000, 800), 50),
                                     ((4000, 300), 100), ((64, 64), 64), ((3, 1000), 3), ((777, 5), 5)])
def test_cpqr_matches_oracle(lr, oracle, shape, k):
    a = inputs.synthetic_np(inputs.scaled(inputs.CONFIGS["c4"], shape[0], shape[1], width=min(shape), k=k))
    ctx = lr.default_context()
    ctx.reset_stats()
    g = lr.cpqr_partial(a, k)
    o = oracle.cpqr(a, k)
    assert np.array_equal(g.pivots, o["pivots"])
    assert rel(g.s, o["s"]) <= TOL and rel(g.q, o["q"]) <= TOL
    st = ctx.stats()
    assert st["cpqr_steps"] == k
    # cpqr.hpp:78-84: the exact-norm recomputes happen at the same (step, column) pairs
    assert st["norm_recomputes"] == o["recomputes"], (st["norm_recomputes"], o["recomputes"])


def test_cpqr_validation(lr, oracle):
    a = oracle.gaussian_matrix(4, 4, 1)
    for k in (0, 5):
        with pytest.raises(ValueError, match="out of range"):
            lr.cpqr_partial(a, k)
    bad = a.copy(); bad[2, 2] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        lr.cpqr_partial(bad, 2)


# ------------------------------------------------------------------ coefficient solve
@pytest.mark.parametrize("kind,esc,ridge", [(0, 1, 0.0), (0, 0, 0.0), (1, 0, 0.0), (2, 0, 0.3)])
def test_coeff_solve_strategies(lr, oracle, kind, esc, ridge):
    s11 = np.triu(oracle.gaussian_matrix(40, 40, 23) + 6.0 * np.eye(40))
    s12 = oracle.gaussian_matrix(40, 333, 24)
    strat = lr.SolveStrategy(kind, 1e-12, ridge, bool(esc))
    t = lr.stabilized_coeff_solve(s11, s12, strat)
    assert rel(t, oracle.coeff_solve(s11, s12, kind, 1e-12, ridge, esc)) <= 1e-10


def test_coeff_solve_edge_cases(lr, oracle):
    s11 = np.zeros((2, 2)); s11[0, 0] = 1.0  # test_solve.cpp:29-38
    t = lr.stabilized_coeff_solve(s11, np.array([[1.0], [0.0]]), lr.SolveStrategy.back_substitution())
    assert t[0, 0] == pytest.approx(1.0) and t[1, 0] == 0.0
    with pytest.raises(lr.SingularityError) as e:  # :40-51
        lr.stabilized_coeff_solve(s11, np.array([[1.0], [0.5]]), lr.SolveStrategy.back_substitution())
    assert e.value.index() == 1
    s11 = np.array([[1.0, 0.5], [0.0, 1e-12]])  # :68-78 escalation == pinv path
    s12 = oracle.gaussian_matrix(2, 2, 8)
    a = lr.stabilized_coeff_solve(s11, s12)
    b = lr.stabilized_coeff_solve(s11, s12, lr.SolveStrategy.truncated_pinv())
    assert np.array_equal(a, b)
    assert lr.default_context().stats()["solve_escalated"] == 1
    t = lr.stabilized_coeff_solve(np.eye(3), np.zeros((3, 0)))  # :112-118
    assert t.shape == (3, 0)
    with pytest.raises(ValueError, match="upper triangular"):
        lr.stabilized_coeff_solve(oracle.gaussian_matrix(3, 3, 2), np.eye(3))
    with pytest.raises(ValueError):
        lr.stabilized_coeff_solve(oracle.gaussian_matrix(3, 2, 1), np.eye(3))


# ------------------------------------------------------------------ SVD / pinv
@pytest.mark.parametrize("shape", [(9, 6), (5, 12), (8, 8), (300, 40), (40, 300)])
def test_svd_pinv_match_oracle(lr, oracle, shape):
    a = oracle.gaussian_matrix(*shape, 11)
    s = lr.svd(a)
    _, so, _ = oracle.svd(a)
    assert rel(s.sigma, so) <= 1e-12
    r = min(shape)
    assert np.linalg.norm(s.u.T @ s.u - np.eye(r)) <= 1e-12 * r
    assert np.linalg.norm(a - (s.u * s.sigma) @ s.v.T) <= 1e-12 * np.linalg.norm(a)
    assert rel(lr.pinv(a), oracle.pinv(a)) <= TOL


def test_pinv_truncation_and_validation(lr):
    a = np.zeros((2, 2)); a[0, 0] = 2.0  # test_svd.cpp:85-91
    p = lr.pinv(a)
    assert p[0, 0] == pytest.approx(0.5) and abs(p[0, 1]) + abs(p[1, 0]) + abs(p[1, 1]) <= 1e-14
    for thr in (0.0, 1.5):
        with pytest.raises(ValueError, match="threshold"):
            lr.pinv(np.eye(3), thr)


# ------------------------------------------------------------------ ID / CUR against the reference fixtures
def test_id_column_golden(lr, gold):
    cid = lr.id_column(gold["id_a"], int(gold["id_k"]))
    assert np.array_equal(cid.pivots, gold["id_piv"])
    assert rel(cid.coeff, gold["id_coeff"]) <= TOL


def test_randomized_id_golden(lr, gold):
    cfg = lr.SketchConfig(oversample=int(gold["rid_p"]), seed=int(gold["rid_seed"]))
    cid = lr.randomized_id(gold["rid_a"], int(gold["rid_k"]), cfg)
    assert np.array_equal(cid.pivots, gold["rid_piv"])
    assert rel(cid.coeff, gold["rid_coeff"]) <= TOL


@pytest.mark.parametrize("mode", [0, 1])
def test_randomized_cur_golden(lr, gold, mode):
    a = gold["rcur_a"]
    cfg = lr.SketchConfig(oversample=int(gold["rcur_p"]), seed=int(gold["rcur_seed"]))
    cur, ts = lr.randomized_cur(a, int(gold["rcur_k"]), cfg, u_mode=mode, return_tsid=True)
    assert np.array_equal(cur.col_pivots, gold[f"rcur{mode}_col_pivots"])
    assert np.array_equal(cur.row_pivots, gold[f"rcur{mode}_row_pivots"])
    assert np.array_equal(cur.c, gold[f"rcur{mode}_c"]) and np.array_equal(cur.r, gold[f"rcur{mode}_r"])
    assert np.array_equal(ts.skeleton, gold["rcur_skeleton"])
    assert rel(cur.u, gold[f"rcur{mode}_u"]) <= TOL
    assert rel(ts.col_id.coeff, gold["rcur_col_coeff"]) <= TOL
    assert rel(ts.row_id.coeff, gold["rcur_row_coeff"]) <= TOL


def test_cur_id_golden(lr, gold):
    cur = lr.cur_id(gold["cur_a"], int(gold["cur_k"]), u_mode=lr.U_CPINV_A_RPINV)
    assert np.array_equal(cur.col_pivots, gold["cur_col_pivots"])
    assert np.array_equal(cur.row_pivots, gold["cur_row_pivots"])
    assert rel(cur.u, gold["cur_u"]) <= TOL


def test_randomized_cur_is_bitwise_repeatable(lr, oracle):  # test_sketch.cpp:170-183
    a = inputs.synthetic_np(inputs.scaled(inputs.CONFIGS["c4"], 600, 700, width=300, k=60))
    cfg = lr.SketchConfig(seed=17)
    c1 = lr.randomized_cur(a, 60, cfg, u_mode=1)
    c2 = lr.randomized_cur(a, 60, cfg, u_mode=1)
    for f in ("c", "u", "r", "col_pivots", "row_pivots"):
        assert np.array_equal(getattr(c1, f), getattr(c2, f))


def test_exact_rank_recovery(lr, oracle):  # test_sketch.cpp:139-146, test_cur.cpp:19-23
    a = oracle.gaussian_matrix(50, 5, 91) @ oracle.gaussian_matrix(5, 35, 1091)
    cid = lr.randomized_id(a, 5, lr.SketchConfig(seed=7))
    assert np.linalg.norm(a - lr.reconstruct(a, cid)) <= 1e-8 * np.linalg.norm(a)
    cur = lr.randomized_cur(a, 5, lr.SketchConfig(seed=7))
    assert np.linalg.norm(a - lr.reconstruct(cur)) <= 1e-8 * np.linalg.norm(a)


def test_error_kernel_matches_oracle(lr, oracle, gold):
    a = gold["rcur_a"]
    cur = lr.randomized_cur(a, 40, lr.SketchConfig(seed=7), u_mode=1)
    e = lr.cur_error_fro(a, cur)
    o = oracle.cur_error_fro(a, cur.c, cur.u, cur.r)
    assert e[0] == pytest.approx(o[0], rel=1e-10) and e[1] == pytest.approx(o[1], rel=1e-13)


def test_validation_messages(lr, oracle):
    a = oracle.gaussian_matrix(6, 9, 2)
    with pytest.raises(ValueError, match="randomized_id: rank"):
        lr.randomized_id(a, 0)
    with pytest.raises(ValueError, match="sample count"):
        lr.randomized_id(a, 5, lr.SketchConfig(oversample=10))
    with pytest.raises(ValueError, match="q must be nonnegative"):
        lr.randomized_id(a, 2, lr.SketchConfig(power=-1))


# ------------------------------------------------------------------ power iterations
@pytest.mark.parametrize("q,reorth", [(1, True), (2, True), (1, False)])
def test_randomized_id_power_matches_oracle(lr, oracle, q, reorth):
    """sketch.hpp:148-164: identical pivots and T within 1e-10 (the GPU's
    orthonormal bases may differ from Householder's by signs, which leaves the
    row space, pivots and T unchanged)."""
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 1500, 1200, width=400, k=60)
    a = inputs.synthetic_np(cfg)
    cid = lr.randomized_id(a, 60, lr.SketchConfig(oversample=10, seed=5, power=q, reorthonormalize=reorth))
    piv, coeff = oracle.randomized_id_power(a, 60, 10, q, reorth, 5)
    assert np.array_equal(cid.pivots, piv)
    assert rel(cid.coeff, coeff) <= TOL


def test_randomized_cur_power_matches_oracle_both_engines(lr, oracle):
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 2000, 1600, width=512, k=80)
    a = inputs.synthetic_np(cfg)
    piv, _ = oracle.randomized_id_power(a, 80, 10, 1, True, 2)
    ctx = lr.default_context()
    for mode in (ctx.GEMM_DMMA, ctx.GEMM_OZAKI_INT8):
        ctx.set_gemm_mode(mode)
        try:
            cur = lr.randomized_cur(a, 80, lr.SketchConfig(oversample=10, seed=2, power=1), u_mode=lr.U_CPINV_A_RPINV)
        finally:
            ctx.set_gemm_mode(ctx.GEMM_DMMA)
        assert np.array_equal(cur.col_pivots, piv)


def test_power_rank_deficient_sample_shrinks(lr, oracle):
    """orth_rows drops numerically dependent rows (svd.hpp:226-231): a rank-20
    matrix with l = 30 leaves a 20-row sample, so k = 25 collapses (sketch.hpp:207-212)
    while k = 15 runs the Householder fallback and matches the oracle."""
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 300, 200, width=20, k=15)
    a = inputs.synthetic_np(cfg)
    cid = lr.randomized_id(a, 15, lr.SketchConfig(oversample=15, seed=1, power=1))
    piv, coeff = oracle.randomized_id_power(a, 15, 15, 1, True, 1)
    assert np.array_equal(cid.pivots[:15], piv[:15])
    with pytest.raises(RuntimeError, match="collapsed"):
        lr.randomized_id(a, 25, lr.SketchConfig(oversample=5, seed=1, power=1))


def test_sketch_power_rows_span_the_oracle_sample(lr, oracle):
    """The sample itself: same row count; the GPU rows span the oracle's row
    space (orthonormal bases agree up to an orthogonal k x k factor)."""
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 800, 700, width=200, k=40)
    a = inputs.synthetic_np(cfg)
    g = lr.sketch_power(a, 50, 1, True, 4).y
    o = oracle.sketch_power(a, 50, 1, True, 4)
    assert g.shape == o.shape
    # q = 0 is exactly the Gaussian sketch (test_sketch.cpp:94-99)
    assert np.array_equal(lr.sketch_power(a, 50, 0, True, 4).y, lr.sketch_gaussian(a, 50, 4).y)
    # both end with Y = Z A for orthonormal Z; project o onto g's row space
    qg, _ = np.linalg.qr(g.T)
    resid = o.T - qg @ (qg.T @ o.T)
    assert np.linalg.norm(resid) <= 1e-10 * np.linalg.norm(o)


# ------------------------------------------------------------------ SRFT sketch
@pytest.mark.parametrize("m", [1024, 1000])
def test_sketch_srft_matches_oracle(lr, oracle, m):
    """sketch.hpp:110-143: the GPU contracts A with the SRFT operator on the
    tensor cores; the reference uses the fast Hartley transform when m is a
    power of two (same operator, roundoff-level differences)."""
    cfg = inputs.scaled(inputs.CONFIGS["c4"], m, 700, width=300, k=50)
    a = inputs.synthetic_np(cfg)
    y = lr.sketch_srft(a, 100, 11).y
    assert rel(y, oracle.sketch_srft(a, 100, 11)) <= 1e-12
    cid = lr.randomized_id(a, 50, lr.SketchConfig(kind=lr.SketchKind.Srft, seed=11))
    piv, coeff = oracle.randomized_id_cfg(a, 50, kind=1, seed=11)
    assert np.array_equal(cid.pivots, piv) and rel(cid.coeff, coeff) <= TOL
    cur = lr.randomized_cur(a, 50, lr.SketchConfig(kind=lr.SketchKind.Srft, srft_samples=80, power=1, seed=2),
                            u_mode=lr.U_CPINV_A_RPINV)
    piv2, _ = oracle.randomized_id_cfg(a, 50, kind=1, srft_samples=80, q=1, seed=2)
    assert np.array_equal(cur.col_pivots, piv2)


# ------------------------------------------------------------------ randomized SVD
@pytest.mark.parametrize("kw", [dict(), dict(power=1), dict(kind=1, seed=5)])
def test_randomized_svd_matches_oracle(lr, oracle, kw):
    """sketch.hpp:238-254: sigma within 1e-10; U and V columns equal up to sign
    (the GPU's orthonormal sample basis may differ from Householder's by signs)."""
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 900, 700, width=300, k=40)
    a = inputs.synthetic_np(cfg)
    sk = lr.SketchConfig(kind=kw.get("kind", 0), power=kw.get("power", 0), seed=kw.get("seed", 1))
    g = lr.randomized_svd(a, 30, sk)
    uo, so, vo = oracle.randomized_svd(a, 30, kind=sk.kind, q=sk.power, seed=sk.seed)
    assert rel(g.sigma, so) <= TOL
    sgn = np.sign(np.sum(g.u * uo, axis=0))
    assert rel(g.u * sgn, uo) <= 1e-9 and rel(g.v * sgn, vo) <= 1e-9


def _ordered_product(om, a):
    """operator * a summed in ascending k as fl(acc + fl(p q)): a host triple loop."""
    y = np.zeros((om.shape[0], a.shape[1]))
    for k in range(om.shape[1]):
        y = y + np.outer(om[:, k], a[k, :])  # elementwise IEEE products, then one rounding per add
    return y


@pytest.mark.parametrize("m,ell,n", [(48, 12, 10), (100, 30, 7), (777, 40, 33)])
def test_srft_dense_fallback_bitwise(lr, oracle, m, ell, n):
    """test_sketch.cpp:76-81: for non-power-of-two m the reference's sketch_srft IS the
    dense product srft_operator(m, l, s) * a (sketch.hpp:137-141), and the test demands
    bitwise equality with that host product.  The GPU reproduces the product's
    arithmetic (ascending k, no FMA) on the library's own operator; against the
    oracle's operator (host libm cos/sin) the sample agrees to roundoff."""
    a = oracle.gaussian_matrix(m, n, m + n)
    y = lr.sketch_srft(a, ell, 8).y
    om = lr.srft_operator(m, ell, 8)
    assert np.array_equal(y, _ordered_product(om, a))
    assert rel(y, oracle.sketch_srft(a, ell, 8)) <= 1e-14


@pytest.mark.parametrize("shape,k", [((250, 37), 37), ((250, 1), 1), ((300, 700), 33), ((512, 1300), 512),
                                     ((500, 3000), 31)])
def test_panel_cpqr_edge_shapes(lr, oracle, shape, k):
    """The delayed-update CPQR (ld 256 / 320 / 512) at ragged panel counts, few
    columns (fewer than one warp per CTA), a single column, a full 512-row panel
    set, and k < one panel: the oracle's pivots, S and Q."""
    a = oracle.gaussian_matrix(shape[0], shape[1], shape[0] + shape[1] + k)
    q = lr.cpqr_partial(a, k)
    o = oracle.cpqr(a, k, want_q=True)
    assert np.array_equal(q.pivots, o["pivots"])
    assert rel(q.s, o["s"]) <= 1e-12 and rel(q.q, o["q"]) <= 1e-12


@pytest.mark.parametrize("shape", [(250, 600), (300, 1000), (500, 1400)])
def test_panel_cpqr_exact_ties(lr, oracle, shape):
    """Exact norm ties on the panel path (logical column swaps): every column
    has a duplicate (negated or not) at a random position, so each pivot's
    twin carries a bitwise-equal norm in any implementation; about a third of
    the columns sit left of k and are moved by the reference's swaps before
    their tie is decided, so the lowest *current* position must win.  k stops
    at rank m: beyond it only rounding noise is left."""
    m, n = shape
    h = n // 2
    rng = np.random.default_rng(m + n)
    g = oracle.gaussian_matrix(m, h, m + h) * (2.0 ** (-rng.random(h) * 8))[None, :]
    pos = rng.permutation(n)
    a = np.zeros((m, n))
    a[:, pos[:h]] = g
    a[:, pos[h:]] = g * np.where(rng.random(h) < 0.5, -1.0, 1.0)[None, :]
    a = np.asfortranarray(a)
    q = lr.cpqr_partial(a, m)
    o = oracle.cpqr(a, m)
    assert np.array_equal(q.pivots, o["pivots"])
    assert rel(q.s, o["s"]) <= 1e-12


def test_panel_cpqr_tie_after_swap(lr):
    """A tie decided by a moved column: v at position 0, -v at position 4, the
    largest column w at position 10.  Step 0 takes w and moves v to position
    10, so step 1's tie goes to -v at position 4 (slot order would pick 0)."""
    m, n = 300, 700
    rng = np.random.default_rng(5)
    a = 0.01 * rng.standard_normal((m, n))
    v = rng.standard_normal(m)
    w = rng.standard_normal(m)
    w -= (w @ v) / (v @ v) * v  # w orthogonal to v: v's residual norm stays exact
    a[:, 0], a[:, 4], a[:, 10] = v, -v, 3.0 * w / np.linalg.norm(w) * np.linalg.norm(v)
    q = lr.cpqr_partial(np.asfortranarray(a), 2)
    assert list(q.pivots[:2]) == [10, 4]


@pytest.mark.parametrize("case", ["zero_columns", "rank_deficient", "all_columns", "sparse_like", "mostly_zero"])
def test_panel_cpqr_degenerate_inputs(lr, oracle, case):
    """Panel CPQR (ld 256 / 320 / 512) on degenerate inputs, against the oracle:
    exact zero columns (norm 0 from the start), a rank-deficient block (norms
    collapse to roundoff and are recomputed), k = n (every slot pivoted, the
    final permutation moves all displaced columns), and a mostly-zero matrix
    like the C^T of the sparse configuration."""
    rng = np.random.default_rng(len(case))
    if case == "zero_columns":
        m, n, k = 300, 900, 300
        a = oracle.gaussian_matrix(m, n, 5)
        a[:, rng.choice(n, 200, replace=False)] = 0.0
    elif case == "rank_deficient":
        m, n, k = 260, 800, 200
        a = oracle.gaussian_matrix(m, 150, 6) @ oracle.gaussian_matrix(150, n, 7)
    elif case == "all_columns":
        m, n, k = 400, 400, 400
        a = oracle.gaussian_matrix(m, n, 8)
    elif case == "sparse_like":
        m, n, k = 300, 3000, 300
        a = np.zeros((m, n))
        for j in range(n):
            rows = rng.choice(m, 3, replace=False)
            a[rows, j] = rng.standard_normal(3)
    else:  # 60 non-zero columns among 2000, k = 150: the last 90 pivots are zero columns, lowest position first
        m, n, k = 300, 2000, 150
        a = np.zeros((m, n))
        a[:, rng.choice(n, 60, replace=False)] = oracle.gaussian_matrix(m, 60, 9)
    a = np.asfortranarray(a)
    q = lr.cpqr_partial(a, k)
    o = oracle.cpqr(a, k)
    if case == "rank_deficient":  # beyond the numerical rank only roundoff is left to pivot on
        assert np.array_equal(q.pivots[:150], o["pivots"][:150])
        assert rel(q.s[:150, :150], o["s"][:150, :150]) <= 1e-10
    else:
        assert np.array_equal(q.pivots, o["pivots"])
        assert rel(q.s, o["s"]) <= 1e-12


@pytest.mark.parametrize("seed", range(8))
def test_panel_cpqr_random_sweep(lr, oracle, seed):
    """Seeded random shapes on the panel path (193 < m <= 512 -> ld 256/320/512,
    ragged n and k, a random share of identically-zero and duplicated columns)
    against the oracle: identical pivots, S to 1e-12."""
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(193, 513))
    n = int(rng.integers(m // 2 + 1, 4 * m))
    a = oracle.gaussian_matrix(m, n, seed) * (2.0 ** rng.uniform(-4, 4, size=n))[None, :]
    nz = int(rng.integers(0, n // 3))
    if nz:
        a[:, rng.choice(n, nz, replace=False)] = 0.0
    nd = int(rng.integers(0, n // 5))
    if nd:
        src = rng.choice(n, nd)
        dst = rng.choice(n, nd)
        a[:, dst] = -a[:, src]
    rank = int(np.linalg.matrix_rank(a))
    k = int(rng.integers(1, max(2, min(m, rank) + 1)))
    a = np.asfortranarray(a)
    q = lr.cpqr_partial(a, k)
    o = oracle.cpqr(a, k)
    assert np.array_equal(q.pivots, o["pivots"])
    assert rel(q.s, o["s"]) <= 1e-12
