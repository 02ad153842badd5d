"""Contraction engine microbenchmark: lr_gemm_tn_d on the DMMA and the Ozaki
INT8 engines (Ozaki timing includes splitting both operands).
    python tools/bench_gemm.py M N K [M N K ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_8447_b200 as lr  # noqa: E402


def run(M, N, K, mode, reps=3):
    ctx = lr.default_context()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.set_gemm_mode(mode)
    P = lr.empty_colmajor(K, M, "cuda")
    P.normal_()
    Q = lr.empty_colmajor(K, N, "cuda")
    for j0 in range(0, N, 4096):  # bounded temporaries
        Q[:, j0:j0 + 4096].normal_()
    out = lr.empty_colmajor(M, N, "cuda")
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = ctx.lib.lr_gemm_tn_d(ctx.h, M, N, K, P.data_ptr(), P.stride(1), Q.data_ptr(), Q.stride(1),
                                  out.data_ptr(), out.stride(1))
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, ctx.lib.lr_last_error()
        best = min(best, e0.elapsed_time(e1))
    ctx.set_gemm_mode(0)
    del P, Q, out
    torch.cuda.empty_cache()
    return {"M": M, "N": N, "K": K, "mode": ["dmma", "ozaki_int8"][mode], "ms": best,
            "TFLOPs_fp64_equiv": 2.0 * M * N * K / (best * 1e-3) / 1e12}


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]] or [510, 65536, 65536, 65536, 500, 65536]
    for i in range(0, len(args), 3):
        for mode in [int(m) for m in os.environ.get("MODES", "0,1").split(",")]:
            print(json.dumps(run(*args[i:i + 3], mode)), flush=True)
