"""GPU parity of the bound-pruned ("lazy") panel CPQR (csrc/cpqr_lazy.cu).

By default the library takes the lazy steps only for sweeps of n >= 32768
columns; LRB_CPQR_LAZY=1 forces them here (the switch is read per call), so
the same shapes the eager kernel is tested on run through the pruned steps,
the retry rounds and panel_finalize_kernel.  The reference semantics
(cpqr.hpp:48-85) are unchanged: identical pivots and exact-norm recompute
counts to the oracle, S and Q within 1e-12; against the eager kernel on the
same device matrix the pivots and recompute counts are identical and S agrees
to roundoff.
"""
import os

import numpy as np
import pytest

from oracle_lib import rel
from paper_1412_8447_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture
def lazy():
    old = os.environ.get("LRB_CPQR_LAZY")
    os.environ["LRB_CPQR_LAZY"] = "1"
    yield
    if old is None:
        del os.environ["LRB_CPQR_LAZY"]
    else:
        os.environ["LRB_CPQR_LAZY"] = old


@pytest.mark.parametrize("shape,k", [((510, 3000), 510), ((500, 4096), 500), ((300, 5000), 300), ((310, 2000), 137),
                                     ((210, 6000), 210), ((256, 1500), 256), ((64, 1000), 64), ((500, 600), 17),
                                     ((320, 700), 1)])
def test_lazy_cpqr_matches_oracle(lr, oracle, lazy, shape, k):
    a = inputs.synthetic_np(inputs.scaled(inputs.CONFIGS["c4"], shape[0], shape[1], width=min(shape), k=k))
    ctx = lr.default_context()
    ctx.reset_stats()
    g = lr.cpqr_partial(a, k)
    o = oracle.cpqr(a, k)
    assert np.array_equal(g.pivots, o["pivots"])
    assert rel(g.s, o["s"]) <= 1e-12 and rel(g.q, o["q"]) <= 1e-12
    assert ctx.stats()["norm_recomputes"] == o["recomputes"]


@pytest.mark.parametrize("seed", range(8))
def test_lazy_cpqr_random_sweep(lr, oracle, lazy, seed):
    """Ragged shapes with identically-zero and (negated) duplicate columns:
    exact norm ties, columns that collapse to zero after their twin is
    pivoted (recomputes), the zero-slot lists."""
    rng = np.random.default_rng(2000 + seed)
    m = int(rng.integers(193, 513))
    n = int(rng.integers(m // 2 + 1, 4 * m))
    a = oracle.gaussian_matrix(m, n, seed) * (2.0 ** rng.uniform(-4, 4, size=n))[None, :]
    nz = int(rng.integers(0, n // 3))
    if nz:
        a[:, rng.choice(n, nz, replace=False)] = 0.0
    nd = int(rng.integers(0, n // 5))
    if nd:
        a[:, rng.choice(n, nd)] = -a[:, rng.choice(n, nd)]
    k = int(rng.integers(1, max(2, min(m, int(np.linalg.matrix_rank(a))) + 1)))
    a = np.asfortranarray(a)
    q = lr.cpqr_partial(a, k)
    o = oracle.cpqr(a, k)
    assert np.array_equal(q.pivots, o["pivots"])
    assert rel(q.s, o["s"]) <= 1e-12


@pytest.mark.parametrize("shape", [(250, 600), (500, 1400)])
def test_lazy_cpqr_exact_ties(lr, oracle, lazy, shape):
    """Every column has a bitwise-equal-norm twin; ties go to the lowest
    current (logical) position, also across skipped columns."""
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


def _device_cpqr(lr, a0, k, lazy_flag):
    import torch
    os.environ["LRB_CPQR_LAZY"] = lazy_flag
    ctx = lr.default_context()
    rows, n = a0.shape
    s = lr.empty_colmajor(k, n, "cuda")
    piv = torch.empty(n, dtype=torch.int64, device="cuda")
    ctx.reset_stats()
    torch.cuda.synchronize()
    rc = ctx.lib.lr_cpqr_partial_d(ctx.h, rows, n, a0.data_ptr(), rows, k, None, s.data_ptr(), piv.data_ptr())
    assert rc == 0, ctx.lib.lr_last_error()
    ctx.synchronize()
    return piv.cpu().numpy(), s.cpu().numpy(), ctx.stats()["norm_recomputes"]


@pytest.mark.parametrize("rows,n,kind", [(510, 40000, "c4"), (500, 32768, "gauss"), (320, 20000, "c4")])
def test_lazy_equals_eager_on_device(lr, rows, n, kind):
    """Same device matrix through both kernels: identical pivots and recompute
    counts, S to roundoff (the C4 sample shape is at the default switch)."""
    import torch
    old = os.environ.get("LRB_CPQR_LAZY")
    try:
        g = torch.Generator(device="cuda").manual_seed(rows + n)
        a0 = lr.empty_colmajor(rows, n, "cuda")
        if kind == "c4":
            w = 1024
            sv = (1.0 + torch.arange(w, dtype=torch.float64, device="cuda") / 50.0) ** -3
            v, _ = torch.linalg.qr(torch.randn(n, w, dtype=torch.float64, device="cuda", generator=g))
            a0.copy_((torch.randn(rows, w, dtype=torch.float64, device="cuda", generator=g) * sv) @ v.T)
        else:
            a0.copy_(torch.randn(rows, n, dtype=torch.float64, device="cuda", generator=g))
        k = rows
        pe, se, re = _device_cpqr(lr, a0, k, "0")
        pl, sl, rl = _device_cpqr(lr, a0, k, "1")
    finally:
        if old is None:
            os.environ.pop("LRB_CPQR_LAZY", None)
        else:
            os.environ["LRB_CPQR_LAZY"] = old
    assert np.array_equal(pl, pe)
    assert re == rl
    assert rel(sl, se) <= 1e-13
