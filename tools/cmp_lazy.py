"""Lazy (bound-pruned) vs eager panel CPQR on the same device matrix.
    python tools/cmp_lazy.py run <out.npz> rows n [c4|gauss|zeros]   (LRB_CPQR_LAZY picks the kernel)
    python tools/cmp_lazy.py cmp <a.npz> <b.npz>
Prints the CPQR time; cmp checks identical pivots / recompute counts and R within 1e-12."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_8447_b200 as lr  # noqa: E402


def make(rows, n, kind, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = lr.empty_colmajor(rows, n, "cuda")
    if kind == "c4":
        w = 1024
        sv = (1.0 + torch.arange(w, dtype=torch.float64, device="cuda") / 50.0) ** -3
        v, _ = torch.linalg.qr(torch.randn(n, w, dtype=torch.float64, device="cuda", generator=g))
        gg = torch.randn(rows, w, dtype=torch.float64, device="cuda", generator=g) * sv
        a.copy_(gg @ v.T)
    elif kind == "zeros":  # sparse-like: most columns identically zero
        x = torch.randn(rows, n, dtype=torch.float64, device="cuda", generator=g)
        x[:, torch.rand(n, device="cuda", generator=g) < 0.85] = 0.0
        a.copy_(x)
    else:
        a.copy_(torch.randn(rows, n, dtype=torch.float64, device="cuda", generator=g))
    return a


def run(out, rows, n, kind):
    ctx = lr.default_context()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    a0 = make(rows, n, kind)
    k = min(rows, n)
    res = {}
    times = []
    for rep in range(3):
        a = a0.clone()
        s = lr.empty_colmajor(k, n, "cuda")
        piv = torch.empty(n, dtype=torch.int64, device="cuda")
        ctx.reset_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        rc = ctx.lib.lr_cpqr_partial_d(ctx.h, rows, n, a.data_ptr(), rows, k, None, s.data_ptr(), piv.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, ctx.lib.lr_last_error()
        times.append(e0.elapsed_time(e1))
        res = {"piv": piv.cpu().numpy(), "s": s.cpu().numpy(), "rec": ctx.stats()["norm_recomputes"]}
    np.savez(out, **res)
    print(json.dumps({"lazy": os.environ.get("LRB_CPQR_LAZY", "1"), "rows": rows, "n": n, "kind": kind,
                      "ms": min(times), "ms_all": times, "recomputes": int(res["rec"])}), flush=True)


def cmp(fa, fb):
    a, b = np.load(fa), np.load(fb)
    same = np.array_equal(a["piv"], b["piv"])
    first = int(np.argmax(a["piv"] != b["piv"])) if not same else -1
    rs = np.linalg.norm(a["s"] - b["s"]) / np.linalg.norm(b["s"])
    print(json.dumps({"a": fa, "b": fb, "pivots_equal": bool(same), "first_diff": first, "rel_s": float(rs),
                      "rec": [int(a["rec"]), int(b["rec"])]}), flush=True)
    return same and rs <= 1e-12 and int(a["rec"]) == int(b["rec"])


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5] if len(sys.argv) > 5 else "gauss")
    else:
        sys.exit(0 if cmp(sys.argv[2], sys.argv[3]) else 1)
