"""GPU: the concurrent CUR tail (row ID of C + R factor on one green-context SM
partition, Q_c and X^T = A^T Q_c on the other; api.cu tsid_cur_split) gives
the sequential path's results: identical pivots and gathers, factors within
roundoff (the Gram products' split-K depends on the partition's SM count)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _run(lr, a, k, split):
    old = os.environ.get("LRB_CUR_SPLIT")
    os.environ["LRB_CUR_SPLIT"] = split
    try:
        ctx = lr.Context(0)
        ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8)
        sk = lr.SketchConfig(oversample=10, seed=7)
        res = {kk: v.cpu().numpy() for kk, v in lr.randomized_cur_device(a, k, sk, u_mode=lr.U_CPINV_A_RPINV,
                                                                        ctx=ctx).items()}
        ctx.synchronize()
        st = ctx.stats()
        ctx.close()
        return res, st
    finally:
        if old is None:
            os.environ.pop("LRB_CUR_SPLIT", None)
        else:
            os.environ["LRB_CUR_SPLIT"] = old


def _rel(x, y):
    return np.linalg.norm(np.asarray(x) - np.asarray(y)) / max(np.linalg.norm(np.asarray(y)), 1e-300)


@pytest.mark.parametrize("k", [300, 500])
def test_concurrent_tail_matches_sequential(lr, k):
    import torch
    from paper_1412_8447_b200 import inputs
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 16384, 16384, width=768, k=k)
    a = inputs.synthetic_torch(cfg, device="cuda", col_block=4096)
    torch.cuda.synchronize()
    seq, st0 = _run(lr, a, k, "0")
    par, st1 = _run(lr, a, k, "56")
    assert st0["concurrent_tail"] == 0 and st1["concurrent_tail"] == 1
    for key in ("col_pivots", "row_pivots", "c", "r", "skeleton"):
        assert np.array_equal(seq[key], par[key]), key
    assert _rel(par["col_coeff"], seq["col_coeff"]) <= 1e-12
    assert _rel(par["row_coeff"], seq["row_coeff"]) <= 1e-12
    assert _rel(par["u"], seq["u"]) <= TOL


def test_concurrent_tail_host_entry(lr):
    """The host-pointer entry (pipelined upload, downloads overlapped with the
    two chains) against the device entry on the same matrix."""
    import torch
    from paper_1412_8447_b200 import inputs
    k = 300
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 16384, 16384, width=768, k=k)
    a = inputs.synthetic_torch(cfg, device="cuda", col_block=4096)
    torch.cuda.synchronize()
    dev, _ = _run(lr, a, k, "56")
    ah = np.asfortranarray(a.cpu().numpy())
    del a
    old = os.environ.get("LRB_CUR_SPLIT")
    os.environ["LRB_CUR_SPLIT"] = "56"
    try:
        ctx = lr.Context(0)
        ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8)
        cur = lr.randomized_cur(ah, k, lr.SketchConfig(oversample=10, seed=7), u_mode=lr.U_CPINV_A_RPINV, ctx=ctx)
        st = ctx.stats()
        ctx.close()
    finally:
        if old is None:
            os.environ.pop("LRB_CUR_SPLIT", None)
        else:
            os.environ["LRB_CUR_SPLIT"] = old
    assert st["concurrent_tail"] == 1
    assert np.array_equal(np.asarray(cur.col_pivots), dev["col_pivots"])
    assert np.array_equal(np.asarray(cur.row_pivots), dev["row_pivots"])
    assert np.array_equal(np.asarray(cur.c), dev["c"]) and np.array_equal(np.asarray(cur.r), dev["r"])
    assert _rel(cur.u, dev["u"]) <= TOL


def test_concurrent_tail_setter_and_automatic_choice(lr):
    """lr_ctx_set_concurrent_tail: an explicit partition size gives the
    sequential results on one context (green contexts rebuilt when the size
    changes); the automatic choice keeps a 16384^2 problem sequential (it
    switches on at m, n >= 32768 with m n >= 2^31 on the INT8 engine: tests/test_gpu_c4_full.py
    runs that against the full-size oracle result) and stays off on the DMMA
    engine."""
    import torch
    from paper_1412_8447_b200 import inputs
    k = 300
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 16384, 16384, width=768, k=k)
    a = inputs.synthetic_torch(cfg, device="cuda", col_block=4096)
    torch.cuda.synchronize()
    ctx = lr.Context(0)
    ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8)
    sk = lr.SketchConfig(oversample=10, seed=7)

    def run():
        r = {kk: v.cpu().numpy() for kk, v in lr.randomized_cur_device(a, k, sk, u_mode=lr.U_CPINV_A_RPINV,
                                                                      ctx=ctx).items()}
        ctx.synchronize()
        return r, ctx.stats()["concurrent_tail"]

    auto, on_auto = run()
    assert on_auto == 0
    res = {}
    for sms in (48, 64, 0):
        ctx.set_concurrent_tail(sms)
        res[sms], on = run()
        assert on == (1 if sms else 0)
    ctx.set_concurrent_tail(-1)
    with pytest.raises(ValueError):
        ctx.set_concurrent_tail(-2)
    ctx.close()
    for sms in (48, 64):
        for key in ("col_pivots", "row_pivots", "c", "r", "skeleton"):
            assert np.array_equal(res[sms][key], res[0][key]), (sms, key)
        assert _rel(res[sms]["u"], res[0]["u"]) <= TOL
    for key in ("col_pivots", "row_pivots", "c", "r", "u"):
        assert np.array_equal(auto[key], res[0][key]), key
