"""BASELINE config 5 (sparse randomized CUR).
The reference is dense-only, so parity is pinned on down-scaled instances
densified through the dense oracle; the full 200000 x 100000 size is checked
through size-independent properties."""
import numpy as np
import pytest

from oracle_lib import rel
from paper_1412_8447_b200 import inputs

pytestmark = pytest.mark.gpu


def densify(row_ptr, col_idx, val, shape):
    m, n = shape
    rp, ci, v = row_ptr.cpu().numpy(), col_idx.cpu().numpy(), val.cpu().numpy()
    a = np.zeros((m, n), order="F")
    for i in range(m):
        a[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    return a


def csc_to_dense(ptr, idx, val, rows, k):
    p, ix, v = ptr.cpu().numpy(), idx.cpu().numpy(), val.cpu().numpy()
    out = np.zeros((rows, k), order="F")
    for t in range(k):
        out[ix[p[t]:p[t + 1]], t] = v[p[t]:p[t + 1]]
    return out


def csr_to_dense(ptr, idx, val, k, cols):
    p, ix, v = ptr.cpu().numpy(), idx.cpu().numpy(), val.cpu().numpy()
    out = np.zeros((k, cols), order="F")
    for t in range(k):
        out[t, ix[p[t]:p[t + 1]]] = v[p[t]:p[t + 1]]
    return out


@pytest.mark.parametrize("mode", [1, 0])
def test_sparse_cur_matches_dense_oracle(lr, oracle, mode):
    m, n, npc, k = 2400, 1200, 12, 40
    row_ptr, col_idx, val = inputs.synthetic_csr_torch(m, n, npc, seed=7)
    a = densify(row_ptr, col_idx, val, (m, n))
    cfg = lr.SketchConfig(oversample=10, seed=3)
    res = lr.randomized_cur_csr_device(row_ptr, col_idx, val, (m, n), k, cfg, u_mode=mode)
    o = oracle.randomized_cur(a, k, 10, 3, u_mode=mode)
    assert np.array_equal(res["col_pivots"].cpu().numpy(), o["col_pivots"])
    assert np.array_equal(res["row_pivots"].cpu().numpy(), o["row_pivots"])
    c = csc_to_dense(res["c_col_ptr"], res["c_row_idx"], res["c_val"], m, k)
    r = csr_to_dense(res["r_row_ptr"], res["r_col_idx"], res["r_val"], k, n)
    assert np.array_equal(c, o["c"]) and np.array_equal(r, o["r"])
    assert rel(res["u"].cpu().numpy(), o["u"]) <= 1e-10
    assert rel(res["col_coeff"][:, : n - k].cpu().numpy(), o["col_coeff"]) <= 1e-10
    e, na = lr.cur_error_fro_csr_device(row_ptr, col_idx, val, (m, n), res)
    eo, nao = oracle.cur_error_fro(a, o["c"], o["u"], o["r"])
    assert na == pytest.approx(nao, rel=1e-13)
    assert e / na == pytest.approx(eo / nao, rel=1e-8)  # ||A||^2 - 2<A,CUR> + ||CUR||^2 (cancellation)


@pytest.mark.slow
def test_sparse_cur_full_size_properties(lr):
    import torch
    m, n, npc, k = 200000, 100000, 100, 300
    row_ptr, col_idx, val = inputs.synthetic_csr_torch(m, n, npc, seed=1412)
    cfg = lr.SketchConfig(oversample=10, seed=1)
    res = lr.randomized_cur_csr_device(row_ptr, col_idx, val, (m, n), k, cfg)
    cp = res["col_pivots"].cpu().numpy()
    rp = res["row_pivots"].cpu().numpy()
    assert np.array_equal(np.sort(cp), np.arange(n)) and np.array_equal(np.sort(rp), np.arange(m))
    # C is exactly the selected columns: each has npc nonzeros with the generator's values
    cptr = res["c_col_ptr"].cpu().numpy()
    assert np.all(np.diff(cptr) == npc)
    res2 = lr.randomized_cur_csr_device(row_ptr, col_idx, val, (m, n), k, cfg)
    for key in ("col_pivots", "row_pivots", "u"):
        assert torch.equal(res[key], res2[key]), key
    nc, nr = int(res["c_col_ptr"][-1]), int(res["r_row_ptr"][-1])
    assert torch.equal(res["c_val"][:nc], res2["c_val"][:nc]) and torch.equal(res["r_val"][:nr], res2["r_val"][:nr])
    e, na = lr.cur_error_fro_csr_device(row_ptr, col_idx, val, (m, n), res)
    assert np.isfinite(e) and 0.0 < e / na <= 1.0
