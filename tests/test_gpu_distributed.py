"""The sharded orchestration (distributed.py) with the B200 DeviceBackend at
world size 1 (the collectives are identities; the multi-rank protocol itself
is covered by tests/test_distributed.py over gloo): same index sets and
factors as the single-GPU pipeline and the CPU oracle."""
import numpy as np
import pytest

from oracle_lib import rel
from paper_1412_8447_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("engine", [0, 1])
def test_sharded_pipeline_on_device_matches_oracle(lr, oracle, engine):
    """engine 1: the Ozaki engine with the shard pinned (lr_ctx_cache_operand)
    so the sketch and A^T Q_c share one residue split."""
    import torch

    from paper_1412_8447_b200 import distributed as D
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 1536, 1280, width=768, k=120)
    a_np = inputs.synthetic_np(cfg)
    a = lr.empty_colmajor(cfg.m, cfg.n, "cuda")
    a.copy_(torch.from_numpy(a_np).cuda())
    be = D.DeviceBackend(lr.default_context(), torch.device("cuda", 0))

    class One:
        world, rank = 1, 0

        def all_gather_cols(self, x):
            return x

        def all_reduce_sum(self, x):
            return x

    ctx = lr.default_context()
    ctx.set_gemm_mode(engine)
    try:
        res = D.randomized_cur_sharded(be, One(), a, 0, cfg.n, cfg.k, oversample=10, seed=5)
        torch.cuda.synchronize()
    finally:
        ctx.set_gemm_mode(0)
        ctx.use_own_stream()
    o = oracle.randomized_cur(a_np, cfg.k, 10, 5, u_mode=1)
    assert np.array_equal(res["col_pivots"].cpu().numpy(), o["col_pivots"])
    assert np.array_equal(res["row_pivots"].cpu().numpy(), o["row_pivots"])
    assert np.array_equal(res["c"].cpu().numpy(), o["c"]) and np.array_equal(res["r"].cpu().numpy(), o["r"])
    assert rel(res["u"].cpu().numpy(), o["u"]) <= 1e-10
    assert rel(res["col_coeff"].cpu().numpy(), o["col_coeff"]) <= 1e-10
    assert rel(res["row_coeff"].cpu().numpy(), o["row_coeff"]) <= 1e-10
