"""Small dense kernels behind U: Cholesky, triangular inverse, CholeskyQR2
(CUDA events around each C-ABI call, device-resident inputs).
    python tools/bench_small.py [rows k]"""
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_8447_b200 as lr  # noqa: E402


def timed(fn, reps=5):
    best, wall = 1e30, 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        wall = min(wall, (time.perf_counter() - t0) * 1e3)
        best = min(best, e0.elapsed_time(e1))
    return round(best, 4), round(wall, 4)


def main(rows, k):
    ctx = lr.default_context()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    x = lr.empty_colmajor(rows, k, "cuda")
    x.normal_()
    g0 = (x.T @ x).contiguous().T.contiguous().T  # column-major k x k
    g = lr.empty_colmajor(k, k, "cuda")
    r = lr.empty_colmajor(k, k, "cuda")
    ri = lr.empty_colmajor(k, k, "cuda")
    ok = ctypes.c_int(0)

    def chol():
        g.copy_(g0)
        assert ctx.lib.lr_cholesky_upper_d(ctx.h, k, g.data_ptr(), g.stride(1)) == 0

    def inv():
        assert ctx.lib.lr_tri_upper_inverse_d(ctx.h, k, g.data_ptr(), g.stride(1), ri.data_ptr(), ri.stride(1)) == 0

    def cq2():
        assert ctx.lib.lr_cholqr2_d(ctx.h, rows, k, x.data_ptr(), x.stride(1), r.data_ptr(), ri.data_ptr(),
                                    ctypes.byref(ok)) == 0

    for name, fn in (("cholesky_upper", chol), ("tri_upper_inverse(abi)", inv), ("cholqr2", cq2)):
        dev, wall = timed(fn)
        print(json.dumps({"op": name, "rows": rows, "k": k, "device_ms": dev, "wall_ms": wall}), flush=True)
    for gm in (0, 1):
        ctx.set_gemm_mode(gm)
        dev, wall = timed(cq2)
        print(json.dumps({"op": "cholqr2", "gemm_mode": gm, "device_ms": dev, "wall_ms": wall}), flush=True)
    ctx.set_gemm_mode(0)


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:]] or [65536, 500]
    main(a[0], a[1])
