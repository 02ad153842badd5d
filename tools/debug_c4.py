"""Stage-timed C4 CURs back to back (debugging aid): host wall time per call
and the library's per-stage device times."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_8447_b200 as lr  # noqa: E402
from paper_1412_8447_b200 import inputs  # noqa: E402

mode = int(os.environ.get("GEMM_MODE", "1"))
cfg = inputs.CONFIGS["c4"]
ctx = lr.Context(0)
lr.lowrank._default = ctx
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ctx.set_gemm_mode(mode)
a = inputs.synthetic_torch(cfg, col_block=8192)
sk = lr.SketchConfig(oversample=cfg.oversample, seed=cfg.sketch_seed)
out = None
for it in range(int(os.environ.get("CALLS", "4"))):
    ctx.reset_stats()
    ctx.enable_timing(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = lr.randomized_cur_device(a, cfg.k, sk, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx, out=out)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rep = ctx.stage_report()
    ctx.enable_timing(False)
    print(json.dumps({"call": it, "host_ms": round(1e3 * (t1 - t0), 2),
                      "stages": {k: round(v["ms"], 2) for k, v in rep.items()}}), flush=True)
