"""BASELINE configs[3] at FULL size (65536 x 65536, k = 500, p = 10,
U = C^+ A R^+) on the GPU against the CPU oracle's full-size run.

The golden fixture tests/golden/c4_full.npz comes from
tools/c4_full_oracle.py (run on a GPU box: A built on the GPU with plain
torch, copied to host, hashed, and factored by the oracle -- the C
restatement of sketch.hpp:227-234 + lowrank_main.cpp:215 -- on all host
cores).  This test rebuilds A the same way, checks its SHA-256, and runs the
randomized CUR on BOTH contraction engines (the Ozaki-II INT8 engine that
bench.py times and the FP64 DMMA engine):

  * column and row index sets identical to the oracle's;
  * C, R and the skeleton bit-exact gathers of A;
  * U within 1e-10 relative of the oracle's;
  * T (column ID, k x (n-k)) and T (row ID, k x (m-k)) within 1e-10
    relative through size-independent checksums: Frobenius norm, per-column
    2-norms, and two seeded projections T g and h^T T;
  * ||A - CUR||_F / ||A||_F within 1e-10 relative of the oracle's;
  * the exact-norm recompute count (cpqr.hpp:78-84) equal to the oracle's.
"""
import os

import numpy as np
import pytest

from oracle_lib import rel
from paper_1412_8447_b200 import inputs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLD = os.path.join(os.path.dirname(__file__), "golden", "c4_full.npz")
TOL = 1e-10


@pytest.fixture(scope="module")
def gold():
    if not os.path.exists(GOLD):
        pytest.skip("tests/golden/c4_full.npz absent (tools/c4_full_oracle.py makes it)")
    return dict(np.load(GOLD))


@pytest.fixture(scope="module")
def c4_matrix(gold):
    import torch
    if torch.cuda.mem_get_info()[0] < 120e9:
        pytest.skip("needs ~120 GB of free HBM (A + the Ozaki residue planes)")
    cfg = inputs.CONFIGS["c4"]
    a = inputs.synthetic_torch(cfg, device="cuda", col_block=8192)
    host = np.empty((cfg.m, cfg.n), order="F")
    ht = torch.from_numpy(host)
    for j0 in range(0, cfg.n, 4096):
        ht[:, j0:j0 + 4096].copy_(a[:, j0:j0 + 4096])
    digest = inputs.sha256_colblocks(host)
    del ht, host
    assert digest == str(gold["a_sha256"]), "the regenerated C4 matrix differs from the golden run's input"
    yield a
    # hand the ~100 GB (A, its residue planes) back for the later full-size tests
    del a
    import paper_1412_8447_b200 as lr
    lr.default_context().release_workspace()
    torch.cuda.empty_cache()


def _checks(t, gold, prefix):
    k, c = t.shape
    g = inputs.gaussian_np(c, 1, int(gold["proj_seed_g"]))[:, 0]
    h = inputs.gaussian_np(k, 1, int(gold["proj_seed_h"]))[:, 0]
    return {"fro": np.linalg.norm(t), "colnorms": np.linalg.norm(t, axis=0), "tg": t @ g, "ht": h @ t}


@pytest.mark.parametrize("engine", ["ozaki", "dmma"])
def test_c4_full_size_vs_oracle(lr, gold, c4_matrix, engine):
    import torch
    a = c4_matrix
    k = int(gold["k"])
    ctx = lr.default_context()
    ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8 if engine == "ozaki" else ctx.GEMM_DMMA)
    try:
        ctx.reset_stats()
        sk = lr.SketchConfig(oversample=int(gold["oversample"]), seed=int(gold["sketch_seed"]))
        out = lr.randomized_cur_device(a, k, sk, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx)
        torch.cuda.synchronize()
        stats = ctx.stats()
    finally:
        ctx.set_gemm_mode(ctx.GEMM_DMMA)

    cp = out["col_pivots"].cpu().numpy()
    rp = out["row_pivots"].cpu().numpy()
    assert np.array_equal(cp, gold["col_pivots"]), f"{engine}: column index set differs"
    assert np.array_equal(rp, gold["row_pivots"]), f"{engine}: row index set differs"
    J, I = out["col_pivots"][:k], out["row_pivots"][:k]
    assert torch.equal(out["c"], a[:, J])
    assert torch.equal(out["r"], a[I, :])
    assert torch.equal(out["skeleton"], a[I][:, J])
    assert np.array_equal(out["skeleton"].cpu().numpy(), gold["skeleton"])
    assert rel(out["u"].cpu().numpy(), gold["u"]) <= TOL

    for key, prefix in (("col_coeff", "tcol"), ("row_coeff", "trow")):
        t = out[key].cpu().numpy()
        ck = _checks(t, gold, prefix)
        assert abs(ck["fro"] - gold[f"{prefix}_fro"]) <= TOL * gold[f"{prefix}_fro"], key
        for name in ("colnorms", "tg", "ht"):
            assert rel(ck[name], gold[f"{prefix}_{name}"]) <= TOL, (key, name)

    e, na = lr.cur_error_fro_device(a, out, ctx=ctx)
    assert e / na == pytest.approx(float(gold["err"]) / float(gold["na"]), rel=TOL)
    assert stats["norm_recomputes"] == int(gold["recomputes_y"]) + int(gold["recomputes_ct"]), \
        (stats["norm_recomputes"], int(gold["recomputes_y"]), int(gold["recomputes_ct"]))
    # the automatic tail schedule: concurrent chains on the INT8 engine at this size, sequential on DMMA
    if "LRB_CUR_SPLIT" not in os.environ:
        assert stats["concurrent_tail"] == (1 if engine == "ozaki" else 0)


def test_c4_full_size_verifiers(lr, gold, c4_matrix):
    """verify.hpp's Lemma 1 and Corollary at 65536^2 on the GPU (block Krylov
    spectral norms of the never-formed 34 GB residuals): the bounds hold, and
    each spectral norm sits below the matching Frobenius norm."""
    import torch
    a = c4_matrix
    k = int(gold["k"])
    ctx = lr.default_context()
    sk = lr.SketchConfig(oversample=int(gold["oversample"]), seed=int(gold["sketch_seed"]))
    out = lr.randomized_cur_device(a, k, sk, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx)
    torch.cuda.synchronize()
    l1 = lr.verify_lemma1_device(a, k, out["col_pivots"], out["col_coeff"], out["row_pivots"], out["row_coeff"],
                                 out["u"])
    assert l1["holds"] and 0.0 < l1["lhs"] <= l1["rhs"] * (1 + 1e-8)
    e, na = lr.cur_error_fro_device(a, out, ctx=ctx)
    assert l1["lhs"] <= e * (1 + 1e-12)  # ||.||_2 <= ||.||_F
    co = lr.verify_corollary_device(a, k, out["col_pivots"], out["col_coeff"], out["u"])
    assert co["holds"] and co["e_norm"] == pytest.approx(l1["e_norm"], rel=1e-10)
    assert co["lhs"] == pytest.approx(l1["lhs"], rel=1e-10)
    print(f"C4 lemma1 {l1}  corollary {co}")


def test_c4_full_size_sharded_protocol_8_shards(lr, gold, c4_matrix):
    """The column-sharded pipeline (lr_randomized_cur_sharded_d) at full C4 size
    with its CPQRs run as 8 column blocks (shard emulation: each step the 8
    blocks' pivot candidates are gathered and every block applies the winner's
    reflector to its own columns -- the multi-GPU protocol on one GPU, kernels
    in sequence): the oracle's index sets, U, T checksums and error."""
    import torch

    from paper_1412_8447_b200 import distributed as D
    a = c4_matrix
    k = int(gold["k"])
    ctx = lr.default_context()
    ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8)
    D.set_shard_emulation(ctx, 8)
    try:
        ctx.reset_stats()
        sk = lr.SketchConfig(oversample=int(gold["oversample"]), seed=int(gold["sketch_seed"]))
        out = D.randomized_cur_sharded_device(ctx, a, 0, a.shape[1], k, sk)
        torch.cuda.synchronize()
        stats = ctx.stats()
    finally:
        D.set_shard_emulation(ctx, 0)
        ctx.set_gemm_mode(ctx.GEMM_DMMA)
    assert np.array_equal(out["col_pivots"].cpu().numpy(), gold["col_pivots"])
    assert np.array_equal(out["row_pivots"].cpu().numpy(), gold["row_pivots"])
    assert rel(out["u"].cpu().numpy(), gold["u"]) <= TOL
    for key, prefix in (("col_coeff", "tcol"), ("row_coeff", "trow")):
        ck = _checks(out[key].cpu().numpy(), gold, prefix)
        for name in ("colnorms", "tg", "ht"):
            assert rel(ck[name], gold[f"{prefix}_{name}"]) <= TOL, (key, name)
    cur = {"c": out["c"], "u": out["u"], "r": out["r_local"]}
    e, na = lr.cur_error_fro_device(a, cur, ctx=ctx)
    assert e / na == pytest.approx(float(gold["err"]) / float(gold["na"]), rel=TOL)
    assert stats["norm_recomputes"] == int(gold["recomputes_y"]) + int(gold["recomputes_ct"])
