"""GPU: the small dense kernels behind the CUR's U (CholeskyQR2 of the C and R
skeletons): blocked Cholesky, triangular inverses, CholeskyQR2 itself, against
numpy on the same inputs.  Tolerances are relative to the conditioning of the
seeded inputs (well conditioned: 1e-12 on residuals)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(lr, a):
    import torch
    t = lr.empty_colmajor(a.shape[0], a.shape[1], "cuda")
    t.copy_(torch.as_tensor(a, device="cuda"))
    torch.cuda.synchronize()
    return t


def _upper_wellcond(k, seed):
    rng = np.random.default_rng(seed)
    r = np.triu(rng.standard_normal((k, k))) / np.sqrt(k)
    r[np.diag_indices(k)] = 1.0 + rng.random(k)
    return np.asfortranarray(r)


@pytest.mark.parametrize("k", [1, 5, 64, 65, 100, 128, 129, 257, 500, 513])
def test_cholesky_upper(lr, k):
    ctx = lr.default_context()
    rng = np.random.default_rng(k)
    x = rng.standard_normal((3 * k + 7, k))
    g = np.asfortranarray(x.T @ x)
    d = _dev(lr, g)
    rc = ctx.lib.lr_cholesky_upper_d(ctx.h, k, d.data_ptr(), d.stride(1))
    assert rc == 0, ctx.lib.lr_last_error()
    ctx.synchronize()
    r = d.cpu().numpy()
    assert np.array_equal(r, np.triu(r))
    assert np.all(np.diag(r) > 0)
    assert np.linalg.norm(r.T @ r - g) <= 1e-12 * np.linalg.norm(g)
    ref = np.linalg.cholesky(g).T
    assert np.linalg.norm(r - ref) <= 1e-10 * np.linalg.norm(ref)


def test_cholesky_upper_reports_failure(lr):
    ctx = lr.default_context()
    k = 200
    g = np.eye(k)
    g[150, 150] = -1.0
    d = _dev(lr, np.asfortranarray(g))
    rc = ctx.lib.lr_cholesky_upper_d(ctx.h, k, d.data_ptr(), d.stride(1))
    assert rc != 0


@pytest.mark.parametrize("k", [1, 7, 64, 65, 127, 128, 200, 500, 512, 513])
def test_tri_upper_inverse(lr, k):
    ctx = lr.default_context()
    r = _upper_wellcond(k, 100 + k)
    d = _dev(lr, r)
    out = lr.empty_colmajor(k, k, "cuda")
    rc = ctx.lib.lr_tri_upper_inverse_d(ctx.h, k, d.data_ptr(), d.stride(1), out.data_ptr(), out.stride(1))
    assert rc == 0, ctx.lib.lr_last_error()
    ctx.synchronize()
    ri = out.cpu().numpy()
    assert np.array_equal(ri, np.triu(ri))
    assert np.linalg.norm(ri @ r - np.eye(k)) <= 1e-12 * k


@pytest.mark.parametrize("rows,k", [(100, 1), (300, 64), (1000, 129), (4096, 500), (2000, 513)])
def test_cholqr2(lr, rows, k):
    ctx = lr.default_context()
    rng = np.random.default_rng(rows + k)
    # moderately conditioned tall matrix (cond ~ 1e3)
    q, _ = np.linalg.qr(rng.standard_normal((rows, k)))
    x = np.asfortranarray((q * np.logspace(0, -3, k)) @ _upper_wellcond(k, k))
    d = _dev(lr, x)
    r = lr.empty_colmajor(k, k, "cuda")
    ri = lr.empty_colmajor(k, k, "cuda")
    ok = ctypes.c_int(-1)
    rc = ctx.lib.lr_cholqr2_d(ctx.h, rows, k, d.data_ptr(), d.stride(1), r.data_ptr(), ri.data_ptr(),
                              ctypes.byref(ok))
    assert rc == 0, ctx.lib.lr_last_error()
    ctx.synchronize()
    assert ok.value == 1
    rh, rih = r.cpu().numpy(), ri.cpu().numpy()
    assert np.array_equal(rh, np.triu(rh))
    qh = x @ rih
    assert np.linalg.norm(qh.T @ qh - np.eye(k)) <= 1e-12 * k
    assert np.linalg.norm(qh @ rh - x) <= 1e-13 * np.linalg.norm(x) * k
