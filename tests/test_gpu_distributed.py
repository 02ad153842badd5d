"""The column-sharded device path (lr_randomized_cur_sharded_d /
lr_cpqr_sharded_d: csrc/shard.cu + csrc/api.cu) on one GPU.

* world size 1, with and without an attached 1-rank NCCL communicator (the
  collectives then really go through NCCL): index sets identical to the CPU
  oracle, C/R/skeleton exact gathers, T/U within 1e-10;
* the multi-rank CPQR logic on one GPU by shard emulation
  (lr_ctx_set_shard_emulation: N column blocks in one process, candidates
  gathered by device copies, every block's step kernel run in sequence -- no
  kernel waits on another): pivots, R rows and every factor BITWISE equal to
  the unsharded run for N = 2, 3, 8 (each column's arithmetic does not depend
  on its owner), recompute counts equal to the oracle's.
The multi-process protocol itself runs over gloo in tests/test_distributed.py."""
import numpy as np
import pytest

from oracle_lib import rel
from paper_1412_8447_b200 import inputs

pytestmark = pytest.mark.gpu
KEYS = ("col_pivots", "row_pivots", "c", "u", "r_local", "col_coeff", "row_coeff", "skeleton")


def _problem(lr, m=1536, n=1280, width=768, k=120):
    import torch
    cfg = inputs.scaled(inputs.CONFIGS["c4"], m, n, width=width, k=k)
    a_np = inputs.synthetic_np(cfg)
    a = lr.empty_colmajor(cfg.m, cfg.n, "cuda")
    a.copy_(torch.from_numpy(a_np).cuda())
    return cfg, a_np, a


def _run(lr, D, a, cfg, engine=0, shards=0, u_mode=None, nccl=False):
    import torch
    ctx = lr.default_context()
    ctx.set_gemm_mode(engine)
    D.set_shard_emulation(ctx, shards)
    try:
        if nccl:
            D.attach_nccl(ctx, world=1, rank=0)
        ctx.reset_stats()
        res = D.randomized_cur_sharded_device(ctx, a, 0, cfg.n, cfg.k, lr.SketchConfig(oversample=10, seed=5),
                                              u_mode=u_mode)
        torch.cuda.synchronize()
        stats = ctx.stats()
    finally:
        if nccl:
            D.detach_nccl(ctx)
        D.set_shard_emulation(ctx, 0)
        ctx.set_gemm_mode(0)
    return {kk: v.cpu().numpy() for kk, v in res.items()}, stats


@pytest.mark.parametrize("engine,u_mode", [(0, 1), (1, 1), (0, 0)])
def test_sharded_cur_device_matches_oracle(lr, oracle, engine, u_mode):
    from paper_1412_8447_b200 import distributed as D
    cfg, a_np, a = _problem(lr)
    res, stats = _run(lr, D, a, cfg, engine=engine, u_mode=u_mode)
    o = oracle.randomized_cur(a_np, cfg.k, 10, 5, u_mode=u_mode)
    assert np.array_equal(res["col_pivots"], o["col_pivots"])
    assert np.array_equal(res["row_pivots"], o["row_pivots"])
    assert np.array_equal(res["c"], o["c"]) and np.array_equal(res["r_local"], o["r"])
    assert np.array_equal(res["skeleton"], o["skeleton"])
    assert rel(res["u"], o["u"]) <= 1e-10
    assert rel(res["col_coeff"], o["col_coeff"]) <= 1e-10
    assert rel(res["row_coeff"], o["row_coeff"]) <= 1e-10
    y = oracle.sketch_gaussian(a_np, cfg.k + 10, 5)
    n_rec = oracle.cpqr(y, cfg.k + 10, want_q=False)["recomputes"] + \
        oracle.cpqr(np.asfortranarray(o["c"].T), cfg.k, want_q=False)["recomputes"]
    assert stats["norm_recomputes"] == n_rec


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_emulated_shards_are_bitwise_identical(lr, shards):
    from paper_1412_8447_b200 import distributed as D
    cfg, _, a = _problem(lr)
    ref, st0 = _run(lr, D, a, cfg)
    got, st1 = _run(lr, D, a, cfg, shards=shards)
    for kk in KEYS:
        assert np.array_equal(ref[kk], got[kk]), kk
    assert st0["norm_recomputes"] == st1["norm_recomputes"]


def test_one_rank_nccl_communicator_is_bitwise_identical(lr):
    """A real (1-rank) NCCL communicator: every exchange goes through
    ncclAllGather / ncclAllReduce; the result equals the communicator-free run."""
    from paper_1412_8447_b200 import distributed as D
    cfg, _, a = _problem(lr, 1024, 1100, 512, 96)
    ref, _ = _run(lr, D, a, cfg)
    got, _ = _run(lr, D, a, cfg, nccl=True)
    for kk in KEYS:
        assert np.array_equal(ref[kk], got[kk]), kk


@pytest.mark.parametrize("shape,k,shards", [((510, 3000), 510, 1), ((510, 3000), 510, 4), ((300, 5000), 137, 3),
                                            ((64, 200), 64, 8), ((40, 9), 9, 8)])
def test_sharded_cpqr_matches_oracle(lr, oracle, shape, k, shards):
    import torch

    from paper_1412_8447_b200 import distributed as D
    a_np = inputs.synthetic_np(inputs.scaled(inputs.CONFIGS["c4"], shape[0], shape[1], width=min(shape), k=k))
    a = lr.empty_colmajor(*shape, "cuda")
    a.copy_(torch.from_numpy(a_np).cuda())
    ctx = lr.default_context()
    D.set_shard_emulation(ctx, shards)
    try:
        ctx.reset_stats()
        piv, s = D.cpqr_sharded_device(ctx, a, 0, shape[1], k)
        torch.cuda.synchronize()
        st = ctx.stats()
    finally:
        D.set_shard_emulation(ctx, 0)
    o = oracle.cpqr(a_np, k, want_q=False)
    assert np.array_equal(piv.cpu().numpy(), o["pivots"])
    assert rel(s.cpu().numpy(), o["s"]) <= 1e-10
    assert st["norm_recomputes"] == o["recomputes"]


def test_sharded_cur_validation(lr):
    import torch

    from paper_1412_8447_b200 import distributed as D
    cfg, a_np, a = _problem(lr, 300, 260, 200, 40)
    bad = a.clone()
    bad[3, 7] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        D.randomized_cur_sharded_device(lr.default_context(), bad, 0, cfg.n, cfg.k)
    with pytest.raises(ValueError):  # block beyond the matrix
        D.randomized_cur_sharded_device(lr.default_context(), a, 10, cfg.n, cfg.k)
    with pytest.raises(NotImplementedError):
        D.randomized_cur_sharded_device(lr.default_context(), a, 0, cfg.n, cfg.k, lr.SketchConfig(power=1))
    torch.cuda.synchronize()


@pytest.mark.parametrize("engine", [0, 1])
def test_sharded_host_entry_matches_device_entry(lr, engine):
    """lr_randomized_cur_sharded (host block, chunked upload overlapped with the
    sketch) gives the device entry's factors: bitwise on the Ozaki engine
    (exact integer products), to roundoff on DMMA (the chunked sketch GEMM may
    pick another split-K)."""
    from paper_1412_8447_b200 import distributed as D
    cfg, a_np, a = _problem(lr, 1536, 1280, 768, 120)
    ref, _ = _run(lr, D, a, cfg, engine=engine)
    ctx = lr.default_context()
    ctx.set_gemm_mode(engine)
    try:
        got = D.randomized_cur_sharded_host(ctx, a_np, 0, cfg.n, cfg.k, lr.SketchConfig(oversample=10, seed=5))
    finally:
        ctx.set_gemm_mode(0)
    for kk in KEYS:
        g = got[kk][:, :ref[kk].shape[1]] if got[kk].ndim == 2 else got[kk]
        if engine == 1 or kk in ("col_pivots", "row_pivots", "c", "r_local", "skeleton"):
            assert np.array_equal(ref[kk], g), kk
        else:
            assert rel(g, ref[kk]) <= 1e-12, kk
