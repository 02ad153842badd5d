"""The Ozaki-II contraction engine (LR_GEMM_OZAKI_INT8: FP64 emulated on the
INT8 tcgen05 tensor cores) against exact and FP64 references, and the CUR
pipeline run on it against the CPU oracle.

Tolerances: the emulated product is exact for the inputs truncated to
beta >= 54 bits relative to each column's largest entry, so per entry
|C - C_exact| <= 2^-beta (max|P_i| sum|Q_j| + max|Q_j| sum|P_i|) (+ one final
rounding); the pipeline keeps the north_star bar (identical index sets,
1e-10 relative factors).
"""
import numpy as np
import pytest

from oracle_lib import rel
from paper_1412_8447_b200 import inputs

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture
def ozaki(lr):
    ctx = lr.default_context()
    ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8)
    try:
        yield ctx
    finally:
        ctx.set_gemm_mode(ctx.GEMM_DMMA)


def _gemm(lr, ctx, P, Q):
    import torch
    K, M = P.shape
    N = Q.shape[1]
    Pc = lr.empty_colmajor(K, M, "cuda"); Pc.copy_(torch.as_tensor(P, device="cuda"))
    Qc = lr.empty_colmajor(K, N, "cuda"); Qc.copy_(torch.as_tensor(Q, device="cuda"))
    out = lr.empty_colmajor(M, N, "cuda")
    torch.cuda.synchronize()  # inputs copied on torch's stream
    rc = ctx.lib.lr_gemm_tn_d(ctx.h, M, N, K, Pc.data_ptr(), Pc.stride(1), Qc.data_ptr(), Qc.stride(1),
                              out.data_ptr(), out.stride(1))
    assert rc == 0, ctx.lib.lr_last_error()
    ctx.synchronize()
    return out.cpu().numpy()


def _exact(P, Q):
    """P^T Q in extended precision (x87 long double, 64-bit significand)."""
    return (P.astype(np.longdouble).T @ Q.astype(np.longdouble))


def _bound(P, Q, beta):
    aP, aQ = np.abs(P), np.abs(Q)
    b = (aP.max(axis=0)[:, None] * aQ.sum(axis=0)[None, :] + aP.sum(axis=0)[:, None] * aQ.max(axis=0)[None, :])
    return 2.0 ** -beta * b


def _beta(K):
    moduli = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]
    log2m = sum(np.log2(moduli))
    return min(int(np.floor((log2m - 1 - np.log2(max(K, 1))) / 2)), 60)


def test_gemm_mode_switch(lr):
    ctx = lr.default_context()
    assert ctx.gemm_mode() == ctx.GEMM_DMMA
    with pytest.raises(ValueError):
        ctx.set_gemm_mode(7)
    ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8)
    assert ctx.gemm_mode() == ctx.GEMM_OZAKI_INT8
    ctx.set_gemm_mode(ctx.GEMM_DMMA)


@pytest.mark.parametrize("M,N,K", [(510, 1000, 777), (128, 256, 128), (5, 7, 3), (300, 260, 4100),
                                   (129, 257, 129), (1, 1, 1), (64, 300, 65536), (33, 70, 20002),
                                   (20, 40, 16384), (210, 1300, 20000), (250, 150, 65536)])
def test_ozaki_gemm_error_bound(lr, ozaki, M, N, K):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    P = rng.standard_normal((K, M))
    Q = rng.standard_normal((K, N))
    out = _gemm(lr, ozaki, P, Q)
    ex = _exact(P, Q)
    err = np.abs(out - ex).astype(np.float64)
    bound = _bound(P, Q, _beta(K)) + np.abs(ex).astype(np.float64) * 2.0 ** -52
    assert np.all(err <= bound)
    # and at least as accurate as the FP64 GEMM overall
    dm = (P.T @ Q)
    assert np.linalg.norm(err) <= 2 * np.linalg.norm((dm - ex).astype(np.float64)) + 1e-300


@pytest.mark.parametrize("K", [1000, 16390])
def test_ozaki_gemm_scaling_and_special_columns(lr, ozaki, K):
    rng = np.random.default_rng(5)
    M, N = 40, 70
    P = rng.standard_normal((K, M))
    Q = rng.standard_normal((K, N))
    P[:, 3] = 0.0                       # zero column
    Q[:, 5] = 0.0
    P[:, 7] *= 2.0 ** 200               # per-column scales far apart
    P[:, 8] *= 2.0 ** -300
    Q[:, 9] *= 2.0 ** 150
    Q[:, 10] *= 2.0 ** -250
    P[::3, 11] *= 1e6                   # dynamic range inside a column
    Q[:, 12] = np.round(Q[:, 12] * 8)   # small integers: exact
    P[:, 13] = np.round(P[:, 13] * 8)
    out = _gemm(lr, ozaki, P, Q)
    ex = _exact(P, Q)
    err = np.abs(out - ex).astype(np.float64)
    bound = _bound(P, Q, _beta(K)) + np.abs(ex).astype(np.float64) * 2.0 ** -52
    assert np.all(err <= bound)
    assert np.all(out[3, :] == 0.0) and np.all(out[:, 5] == 0.0)
    assert out[13, 12] == float(P[:, 13] @ Q[:, 12])  # integer data: exact


@pytest.mark.parametrize("K", [16384, 30002, 65536])
def test_ozaki_fused_split_equals_two_pass(lr, ozaki, K, monkeypatch):
    """The cluster-fused column max + split (one read of X) and the two-pass
    colmax_kernel + split_kernel give bit-identical products, NaN / Inf /
    zero columns included."""
    rng = np.random.default_rng(K)
    P = rng.standard_normal((K, 24))
    Q = rng.standard_normal((K, 37))
    P[:, 2] = 0.0
    P[K // 2, 3] = np.nan
    Q[K - 1, 4] = np.inf
    Q[:, 5] *= 2.0 ** -600
    P[::5, 6] *= 1e8
    monkeypatch.setenv("LRB_SPLIT_FUSED", "1")
    fused = _gemm(lr, ozaki, P, Q)
    monkeypatch.setenv("LRB_SPLIT_FUSED", "0")
    two = _gemm(lr, ozaki, P, Q)
    assert np.array_equal(np.isnan(fused), np.isnan(two))
    assert np.array_equal(np.nan_to_num(fused), np.nan_to_num(two))
    assert np.all(np.isnan(fused[3, :])) and np.all(np.isnan(fused[:, 4]))


def test_ozaki_gemm_deterministic(lr, ozaki):
    rng = np.random.default_rng(9)
    P = rng.standard_normal((3000, 300))
    Q = rng.standard_normal((3000, 500))
    assert np.array_equal(_gemm(lr, ozaki, P, Q), _gemm(lr, ozaki, P, Q))


@pytest.mark.parametrize("shape,k,mode", [((2000, 1500), 50, 1), ((1200, 3000), 100, 0), ((4096, 4096), 500, 1)])
def test_randomized_cur_on_ozaki_matches_oracle(lr, oracle, ozaki, shape, k, mode):
    cfg = inputs.scaled(inputs.CONFIGS["c4"], shape[0], shape[1], width=min(1024, min(shape)), k=k)
    a = inputs.synthetic_np(cfg)
    cur, ts = lr.randomized_cur(a, k, lr.SketchConfig(oversample=10, seed=1), u_mode=mode, return_tsid=True)
    o = oracle.randomized_cur(a, k, 10, 1, u_mode=mode)
    assert np.array_equal(cur.col_pivots, o["col_pivots"])
    assert np.array_equal(cur.row_pivots, o["row_pivots"])
    assert np.array_equal(cur.c, o["c"]) and np.array_equal(cur.r, o["r"])
    assert rel(ts.col_id.coeff, o["col_coeff"]) <= TOL
    assert rel(ts.row_id.coeff, o["row_coeff"]) <= TOL
    assert rel(cur.u, o["u"]) <= TOL
    e, na = lr.cur_error_fro(a, cur)
    eo, nao = oracle.cur_error_fro(a, o["c"], o["u"], o["r"])
    assert e / na == pytest.approx(eo / nao, rel=TOL)


def test_device_cur_ozaki_equals_dmma_indices(lr):
    """Same C4-shaped device problem on both engines: identical skeletons."""
    import torch
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 8192, 8192, width=1024, k=500)
    a = inputs.synthetic_torch(cfg)
    sk = lr.SketchConfig(oversample=10, seed=1)
    ctx = lr.default_context()
    d = lr.randomized_cur_device(a, 500, sk, u_mode=lr.U_CPINV_A_RPINV)
    ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8)
    try:
        z = lr.randomized_cur_device(a, 500, sk, u_mode=lr.U_CPINV_A_RPINV)
    finally:
        ctx.set_gemm_mode(ctx.GEMM_DMMA)
    torch.cuda.synchronize()
    assert torch.equal(d["col_pivots"], z["col_pivots"]) and torch.equal(d["row_pivots"], z["row_pivots"])
    assert torch.equal(d["c"], z["c"]) and torch.equal(d["r"], z["r"])
    du, zu = d["u"].cpu().numpy(), z["u"].cpu().numpy()
    assert rel(zu, du) <= TOL


@pytest.mark.parametrize("engine", [0, 1])
def test_host_pipeline_pinned_outputs_match(lr, oracle, engine):
    """The host entry point uploads A in column chunks overlapped with the
    sketch and copies pinned outputs back on a second stream: same bits as the
    plain (pageable) call, and the oracle's index sets."""
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 3000, 5000, width=1024, k=120)
    a = inputs.synthetic_np(cfg)
    ctx = lr.default_context()
    ctx.set_gemm_mode(engine)
    try:
        sk = lr.SketchConfig(oversample=10, seed=3)
        plain = lr.randomized_cur(a, 120, sk, u_mode=lr.U_CPINV_A_RPINV, return_tsid=True)
        out = lr.pinned_cur_outputs(3000, 5000, 120)
        piped = lr.randomized_cur(a, 120, sk, u_mode=lr.U_CPINV_A_RPINV, return_tsid=True, out=out)
    finally:
        ctx.set_gemm_mode(0)
    (c1, t1), (c2, t2) = plain, piped
    for x, y in [(c1.c, c2.c), (c1.u, c2.u), (c1.r, c2.r), (c1.col_pivots, c2.col_pivots),
                 (c1.row_pivots, c2.row_pivots), (t1.col_id.coeff, t2.col_id.coeff),
                 (t1.row_id.coeff, t2.row_id.coeff), (t1.skeleton, t2.skeleton)]:
        assert np.array_equal(x, y)
    o = oracle.randomized_cur(a, 120, 10, 3, u_mode=1)
    assert np.array_equal(c2.col_pivots, o["col_pivots"]) and np.array_equal(c2.row_pivots, o["row_pivots"])
    assert rel(c2.u, o["u"]) <= TOL


@pytest.mark.parametrize("shape,k", [((333, 257), 1), ((97, 1500), 40), ((1100, 600), 300)])
def test_host_pipeline_edge_shapes_both_engines(lr, oracle, shape, k):
    """Ragged shapes through the host entry point (chunked upload, m not a
    multiple of 16, k = 1, n below one chunk): oracle index sets on both engines."""
    cfg = inputs.scaled(inputs.CONFIGS["c4"], shape[0], shape[1], width=min(shape), k=k)
    a = inputs.synthetic_np(cfg)
    o = oracle.randomized_cur(a, k, 5, 9, u_mode=1)
    ctx = lr.default_context()
    for mode in (ctx.GEMM_DMMA, ctx.GEMM_OZAKI_INT8):
        ctx.set_gemm_mode(mode)
        try:
            cur = lr.randomized_cur(a, k, lr.SketchConfig(oversample=5, seed=9), u_mode=lr.U_CPINV_A_RPINV)
        finally:
            ctx.set_gemm_mode(ctx.GEMM_DMMA)
        assert np.array_equal(cur.col_pivots, o["col_pivots"]) and np.array_equal(cur.row_pivots, o["row_pivots"])
        assert rel(cur.u, o["u"]) <= TOL


def test_host_pipeline_nonfinite_and_strided_input(lr):
    """A NaN in the last upload chunk is reported with the reference's message;
    a strided (lda > m) host matrix gives the same factors as its compact copy."""
    a = np.asfortranarray(np.random.default_rng(3).standard_normal((700, 2100)))
    big = np.zeros((760, 2100), order="F")
    big[:700] = a
    view = big[:700]
    ctx = lr.default_context()
    for mode in (ctx.GEMM_DMMA, ctx.GEMM_OZAKI_INT8):
        ctx.set_gemm_mode(mode)
        try:
            c1 = lr.randomized_cur(a, 30, lr.SketchConfig(seed=4))
            c2 = lr.randomized_cur(view, 30, lr.SketchConfig(seed=4))
            assert np.array_equal(c1.col_pivots, c2.col_pivots) and np.array_equal(c1.u, c2.u)
            bad = a.copy()
            bad[5, 2099] = np.nan
            with pytest.raises(ValueError, match="non-finite"):
                lr.randomized_cur(bad, 30, lr.SketchConfig(seed=4))
        finally:
            ctx.set_gemm_mode(ctx.GEMM_DMMA)


def test_ozaki_gemm_large_k_falls_back(lr, ozaki):
    """K > 2^17 exceeds exact int32 accumulation: the engine runs DMMA instead."""
    rng = np.random.default_rng(2)
    P = rng.standard_normal((140000, 3))
    Q = rng.standard_normal((140000, 2))
    out = _gemm(lr, ozaki, P, Q)
    assert rel(out, P.T @ Q) <= 1e-13


def test_ozaki_gemm_propagates_nonfinite(lr, ozaki):
    """A NaN or Inf in an operand column makes that product column non-finite
    (as an FP64 GEMM would), so the pipeline's finiteness checks still fire."""
    rng = np.random.default_rng(4)
    P = rng.standard_normal((500, 20))
    Q = rng.standard_normal((500, 30))
    P[7, 3] = np.nan
    Q[11, 5] = np.inf
    out = _gemm(lr, ozaki, P, Q)
    assert np.all(np.isnan(out[3, :])) and np.all(~np.isfinite(out[:, 5]))
    keep = np.ones(20, bool)
    keep[3] = False
    assert np.all(np.isfinite(np.delete(out[keep], 5, axis=1)))


def test_ozaki_falls_back_to_dmma_when_planes_do_not_fit(lr, oracle):
    """With too little free HBM for A's residue planes (2 B per byte of A) the
    Ozaki engine runs the FP64 DMMA GEMM instead of failing."""
    import torch
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 12000, 12000, width=1024, k=100)
    a = inputs.synthetic_np(cfg)
    sk = lr.SketchConfig(oversample=10, seed=6)
    ref = lr.randomized_cur(a, 100, sk, u_mode=lr.U_CPINV_A_RPINV)
    ctx = lr.default_context()
    ctx.synchronize()
    torch.cuda.synchronize()
    free = torch.cuda.mem_get_info()[0]
    filler = torch.empty(max(0, free - int(3.2e9)), dtype=torch.uint8, device="cuda")
    try:
        ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8)
        cur = lr.randomized_cur(a, 100, sk, u_mode=lr.U_CPINV_A_RPINV)
    finally:
        ctx.set_gemm_mode(ctx.GEMM_DMMA)
        del filler
        torch.cuda.empty_cache()
    assert np.array_equal(cur.col_pivots, ref.col_pivots) and np.array_equal(cur.row_pivots, ref.row_pivots)
    assert rel(cur.u, ref.u) <= TOL


# ------------------------------------------------------------------ power rounds on the INT8 engine
# Z^T = A Y^T contracts over A's columns: A's cached residue planes enter the tcgen05 GEMM as the
# M-major operand with their column scales folded into Y^T (api.cu power_zt_int8, SURVEY 8f.1 /
# sketch.hpp:148-164).
def _stages(ctx, fn):
    ctx.reset_stats()
    ctx.enable_timing(True)
    try:
        res = fn()
        ctx.synchronize()
        return res, ctx.stage_report()
    finally:
        ctx.enable_timing(False)


@pytest.mark.parametrize("m,n,width,k,q", [(1500, 1200, 400, 60, 1), (1200, 2500, 400, 60, 1),
                                           (2600, 1100, 300, 50, 2), (1024, 4096, 512, 100, 1),
                                           (4099, 3001, 600, 120, 1)])
def test_power_rounds_on_int8_match_oracle(lr, oracle, ozaki, m, n, width, k, q):
    """Identical pivots and T within 1e-10 of the oracle; the stage marks show
    that no A^T was formed (the rounds ran on A's residue planes)."""
    cfg = inputs.scaled(inputs.CONFIGS["c4"], m, n, width=width, k=k)
    a = inputs.synthetic_np(cfg)
    sk = lr.SketchConfig(oversample=10, seed=5, power=q)
    cid, st = _stages(ozaki, lambda: lr.randomized_id(a, k, sk, ctx=ozaki))
    assert "power_zt_gemm" in st and "power_transpose_a" not in st, sorted(st)
    piv, coeff = oracle.randomized_id_power(a, k, 10, q, True, 5)
    assert np.array_equal(cid.pivots, piv)
    assert rel(cid.coeff, coeff) <= TOL


def test_power_round_int8_with_wild_column_scales(lr, ozaki):
    """Columns of A spanning 60 orders of magnitude (the scales folded into
    Y^T span the same range): the INT8 round against the FP64 DMMA round."""
    rng = np.random.default_rng(3)
    m, n, k = 1800, 1500, 40
    cfg = inputs.scaled(inputs.CONFIGS["c4"], m, n, width=300, k=k)
    a = inputs.synthetic_np(cfg) * (10.0 ** rng.integers(-30, 31, size=n))[None, :]
    a = np.asfortranarray(a)
    sk = lr.SketchConfig(oversample=10, seed=9, power=1)
    got, st = _stages(ozaki, lambda: lr.randomized_id(a, k, sk, ctx=ozaki))
    assert "power_transpose_a" not in st
    ozaki.set_gemm_mode(ozaki.GEMM_DMMA)
    ref = lr.randomized_id(a, k, sk, ctx=ozaki)
    assert np.array_equal(got.pivots, ref.pivots)
    assert rel(got.coeff, ref.coeff) <= 1e-9


def test_power_round_int8_randomized_cur_reuses_planes(lr, oracle, ozaki):
    """randomized_cur with q = 1: sketch, both halves of the round and
    A^T Q_c all run on one split of A."""
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 2000, 1600, width=512, k=80)
    a = inputs.synthetic_np(cfg)
    piv, _ = oracle.randomized_id_power(a, 80, 10, 1, True, 2)
    cur, st = _stages(ozaki, lambda: lr.randomized_cur(a, 80, lr.SketchConfig(oversample=10, seed=2, power=1),
                                                       u_mode=lr.U_CPINV_A_RPINV, ctx=ozaki))
    assert "power_transpose_a" not in st
    assert np.array_equal(cur.col_pivots, piv)
