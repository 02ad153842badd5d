#!/usr/bin/env python3
"""Measured dense INT8 tensor-core peak of this B200 (roofline denominator of
the Ozaki-II engine's imma_gemm_kernel), in the same way the driver measures
its bf16 peak for MEASURED_PEAKS.json: a library GEMM (cuBLASLt IMMA through
torch._int_mm, int8 x int8 -> int32) on 8192^3, best of 10 launches (burst)
and back to back for 4 s (sustained, the clock the GEMM holds once the board
is at its power cap).  SM clocks are sampled through NVML during each phase.

    python tools/microbench/int8_peak.py [--out profiles/r02_int8_peak.json]
"""
import argparse
import json
import os
import threading
import time

import torch


def nvml_clock_sampler(stop, samples):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            stop.wait(0.05)
    except Exception:
        pass


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__)))), "profiles", "r02_int8_peak.json"))
    p.add_argument("--n", type=int, default=8192)
    p.add_argument("--seconds", type=float, default=4.0)
    args = p.parse_args()
    n = args.n
    dev = torch.device("cuda", 0)
    a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device=dev)
    b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device=dev).t()  # column-major operand
    ops = 2.0 * n ** 3
    # exactness probe on a slice (the integer product is exact)
    c = torch._int_mm(a[:256], b[:, :256])
    ref = a[:256].to(torch.float64) @ b[:, :256].to(torch.float64)
    assert torch.equal(c.to(torch.float64), ref)
    for _ in range(5):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    stop, s_burst = threading.Event(), []
    th = threading.Thread(target=nvml_clock_sampler, args=(stop, s_burst), daemon=True)
    th.start()
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    stop.set()
    th.join()
    # sustained: back to back for `seconds`
    stop, s_sust = threading.Event(), []
    th = threading.Thread(target=nvml_clock_sampler, args=(stop, s_sust), daemon=True)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < args.seconds:
        for _ in range(20):
            torch._int_mm(a, b)
        iters += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    sust = ops * iters / (e0.elapsed_time(e1) * 1e-3)

    def med(s):
        v = sorted(c for c, _ in s)
        return v[len(v) // 2] if v else None

    rec = {"int8_tops": round(ops / best / 1e12, 1), "int8_tops_sustained": round(sust / 1e12, 1),
           "shape": f"{n}^3 int8 x int8 -> int32 (torch._int_mm, cuBLASLt IMMA)",
           "sm_mhz_median_burst": med(s_burst), "sm_mhz_median_sustained": med(s_sust),
           "throttle_reasons_sustained": sorted({hex(r) for _, r in s_sust}),
           "gpu": torch.cuda.get_device_name(0), "torch": torch.__version__,
           "how": "best of 10 single launches (burst); back to back for %.0f s (sustained); CUDA events" %
                  args.seconds}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
