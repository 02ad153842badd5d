"""The verifiers at scale (verify.hpp:14-166) on the GPU: spectral norms of
residual operators by block Krylov (never materialising the m x n residual)
against the reference semantics -- sigma_1 of a full SVD of the materialised
residual (svd.hpp:185-189), here numpy's -- on instances small enough to
materialise; the lemma / corollary reports field by field."""
import numpy as np
import pytest

from oracle_lib import rel
from paper_1412_8447_b200 import inputs

pytestmark = pytest.mark.gpu
TOL = 1e-10


def dev(lr, x):
    import torch
    t = lr.empty_colmajor(x.shape[0], x.shape[1], "cuda")
    t.copy_(torch.from_numpy(np.asfortranarray(x)).cuda())
    return t


def spec(x):
    return float(np.linalg.norm(x, 2))


@pytest.mark.parametrize("shape,k", [((600, 500), 20), ((300, 900), 0), ((1000, 64), 7)])
def test_residual_norms_match_full_svd(lr, oracle, shape, k):
    m, n = shape
    a = inputs.synthetic_np(inputs.scaled(inputs.CONFIGS["c4"], m, n, width=min(m, n), k=max(k, 1)))
    if k:
        x = oracle.gaussian_matrix(m, k, 3)
        y = oracle.gaussian_matrix(k, n, 4) * 1e-2
        e = a - x @ y
        s, f = lr.residual_norms_device(dev(lr, a), dev(lr, x), dev(lr, y))
    else:
        e = a
        s, f = lr.residual_norms_device(dev(lr, a))
    assert s == pytest.approx(spec(e), rel=1e-12)
    assert f == pytest.approx(np.linalg.norm(e), rel=1e-12)


def _cur(lr, a_np, k):
    import torch
    a = dev(lr, a_np)
    out = lr.randomized_cur_device(a, k, lr.SketchConfig(oversample=10, seed=2), u_mode=lr.U_CPINV_A_RPINV)
    torch.cuda.synchronize()
    return a, out


def _ref_parts(a, out, k):
    """The reference's verify.hpp quantities on materialised numpy matrices."""
    m, n = a.shape
    cp, rp = out["col_pivots"].cpu().numpy(), out["row_pivots"].cpu().numpy()
    cc, rc = out["col_coeff"].cpu().numpy(), out["row_coeff"].cpu().numpy()
    u = out["u"].cpu().numpy()
    c, r = a[:, cp[:k]], a[rp[:k], :]
    v = np.zeros((n, k))  # basis() (id.hpp:21-30)
    for l in range(n):
        if l < k:
            v[cp[l], l] = 1.0
        else:
            v[cp[l], :] = cc[:, l - k]
    w = np.zeros((m, k))
    for l in range(m):
        if l < k:
            w[rp[l], l] = 1.0
        else:
            w[rp[l], :] = rc[:, l - k]
    e = a - c @ v.T
    etilde = a - w @ r
    stack = np.zeros((m, n))  # verify.hpp:108-117
    e_skel = e[rp[:k], :]
    for l in range(k, m):
        stack[rp[l], :] = e[rp[l], :] - rc[:, l - k] @ e_skel
    return dict(c=c, r=r, u=u, v=v, w=w, e=e, etilde=etilde, stack=stack, rc=rc, cp=cp, rp=rp, cc=cc)


def test_lemma1_lemma2_corollary_match_reference_semantics(lr):
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 1024, 900, width=400, k=60)
    a_np = inputs.synthetic_np(cfg)
    k = cfg.k
    a, out = _cur(lr, a_np, k)
    p = _ref_parts(a_np, out, k)
    lhs = spec(a_np - p["c"] @ p["u"] @ p["r"])
    e_norm, et_norm = spec(p["e"]), spec(p["etilde"])

    l1 = lr.verify_lemma1_device(a, k, out["col_pivots"], out["col_coeff"], out["row_pivots"], out["row_coeff"],
                                 out["u"])
    assert l1["e_norm"] == pytest.approx(e_norm, rel=TOL)
    assert l1["etilde_norm"] == pytest.approx(et_norm, rel=TOL)
    assert l1["lhs"] == pytest.approx(lhs, rel=TOL)
    assert l1["rhs"] == pytest.approx(e_norm + et_norm, rel=TOL)
    assert l1["holds"] == (lhs <= (e_norm + et_norm) * (1 + 1e-8)) and l1["holds"]

    l2 = lr.verify_lemma2_device(a, k, out["col_pivots"], out["col_coeff"], out["row_pivots"], out["row_coeff"])
    t_norm = spec(p["rc"])
    assert l2["etilde_norm"] == pytest.approx(et_norm, rel=TOL)
    assert l2["fe_norm"] == pytest.approx(spec(p["stack"]), rel=TOL)
    assert l2["e_norm"] == pytest.approx(e_norm, rel=TOL)
    assert l2["t_norm"] == pytest.approx(t_norm, rel=TOL)
    assert l2["bound_rhs"] == pytest.approx((1 + t_norm) * e_norm, rel=TOL)
    # both paths agree to rounding: the reference's gap and ours are roundoff-sized
    ref_gap = np.abs(p["etilde"] - p["stack"]).max()
    scale = np.abs(a_np).max()
    assert l2["entry_diff"] <= 1e-10 * scale and ref_gap <= 1e-10 * scale
    assert l2["holds"] and l2["bound_holds"]

    co = lr.verify_corollary_device(a, k, out["col_pivots"], out["col_coeff"], out["u"])
    assert co["t_norm"] == pytest.approx(t_norm, rel=TOL)
    assert co["e_norm"] == pytest.approx(e_norm, rel=TOL)
    assert co["lhs"] == pytest.approx(lhs, rel=TOL)
    assert co["bound"] == pytest.approx((2 + t_norm) * e_norm, rel=TOL)
    assert co["ceiling"] == pytest.approx(2 * np.sqrt(k * (cfg.m - k)))
    assert co["holds"]


def test_error_report_and_zero_matrix(lr):
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 500, 400, width=300, k=40)
    a_np = inputs.synthetic_np(cfg)
    a, out = _cur(lr, a_np, cfg.k)
    p = _ref_parts(a_np, out, cfg.k)
    cu = dev(lr, p["c"] @ p["u"])
    rep = lr.error_report_device(a, cu, out["r"])
    diff = a_np - p["c"] @ p["u"] @ p["r"]
    assert rep["abs_spectral"] == pytest.approx(spec(diff), rel=TOL)
    assert rep["rel_spectral"] == pytest.approx(spec(diff) / spec(a_np), rel=TOL)
    assert rep["abs_frob"] == pytest.approx(np.linalg.norm(diff), rel=TOL)
    assert rep["rel_frob"] == pytest.approx(np.linalg.norm(diff) / np.linalg.norm(a_np), rel=TOL)
    assert not rep["rel_is_absolute"]
    z = dev(lr, np.zeros((50, 40)))
    x = dev(lr, np.ones((50, 2)))
    y = dev(lr, np.ones((2, 40)))
    rz = lr.error_report_device(z, x, y)  # verify.hpp:41-44: zero A -> absolute fields
    assert rz["rel_is_absolute"] and rz["rel_frob"] == rz["abs_frob"] == pytest.approx(np.sqrt(50 * 40 * 4.0))
    assert rz["abs_spectral"] == pytest.approx(2.0 * np.sqrt(50 * 40), rel=1e-12)
