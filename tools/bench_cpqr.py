"""CPQR kernel microbenchmark: per-step cost vs trailing width (device data).
    python tools/bench_cpqr.py [rows] [n ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_8447_b200 as lr  # noqa: E402


def run(rows, n, reps=3):
    ctx = lr.default_context()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    a = lr.empty_colmajor(rows, n, "cuda")
    if os.environ.get("SPECTRUM") == "c4":  # sketch of a C4-spectrum matrix: G diag(s) V^T
        w = 1024
        sv = (1.0 + torch.arange(w, dtype=torch.float64, device="cuda") / 50.0) ** -3
        v, _ = torch.linalg.qr(torch.randn(n, w, dtype=torch.float64, device="cuda"))
        g = torch.randn(rows, w, dtype=torch.float64, device="cuda") * sv
        a.copy_(g @ v.T)
        del v, g
    else:
        g = torch.randn(n, rows, dtype=torch.float64, device="cuda")
        a.copy_(g.T)
    k = min(rows, n)
    s = lr.empty_colmajor(k, n, "cuda")
    piv = torch.empty(n, dtype=torch.int64, device="cuda")
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = ctx.lib.lr_cpqr_partial_d(ctx.h, rows, n, a.data_ptr(), rows, k, None, s.data_ptr(), piv.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, ctx.lib.lr_last_error()
        best = min(best, e0.elapsed_time(e1))
    byts = sum(16.0 * (rows - t) * (n - t) + 32.0 * (n - t) for t in range(k))
    st = ctx.stats() if hasattr(ctx, "stats") else {}
    return {"stats": st, "rows": rows, "n": n, "steps": k, "ms": best, "us_per_step": 1e3 * best / k,
            "GBps_alg": byts / (best * 1e-3) / 1e9}


if __name__ == "__main__":
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 510
    ns = [int(x) for x in sys.argv[2:]] or [512, 2048, 8192, 32768, 65536]
    for n in ns:
        print(json.dumps(run(rows, n)), flush=True)
