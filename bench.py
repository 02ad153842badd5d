#!/usr/bin/env python3
"""Benchmark: time-to-CUR for randomized CUR, BASELINE.json configs[3]
(A 65536 x 65536 fp64 = U diag(s) V^T, width 1024, s_j = (1+j/50)^-3,
k = 500, p = 10, U = C^+ A R^+).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c1|c2|c3|c5]

One "step" = one full randomized CUR (sketch -> CPQR(Y) -> T solve -> row ID
on C -> U = C^+ A R^+ and the tsID skeleton) with A resident in HBM
(`value`), and again through the host C ABI with A in pinned host memory and
the factors copied back (`e2e`).  A is 34.4 GB, larger than the 126 MB L2, so
no flush is needed between steps.  Device time = CUDA events on the stream
the library launches on, max over ranks.

The two A-sized contractions run on the Ozaki-II engine by default
(--engine ozaki: FP64 products of inputs rounded to 54 bits per column,
computed exactly on the INT8 tensor cores); --engine
dmma uses the FP64 DMMA GEMM.

--gpus N without torchrun: bench.py re-launches itself under
torch.distributed.run with N ranks (127.0.0.1 rendezvous).  N > 1: the
column-sharded path by default (--mode sharded, strong scaling,
distributed.py); --mode replicas factors one copy of A per rank.

--impl reference: the reference's CPU algorithm (the C restatement in
oracle/, see DESIGN.md for why not oracle/_ref) on ALL host cores, run ONCE
at the full configuration (C4: about 6-10 min on a 16-core host; the line
reports steps = 1 whatever --steps asked).  C1-C3: median of 5 full runs.

--workload c1|c2|c3: BASELINE configs[0..2] (deterministic column ID
1000x800 k=50; deterministic CUR 4000x3000 k=100; randomized column ID
20000^2 k=200 p=10), device-resident, with the measured full-size CPU
oracle run next to them.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M = N = 65536
K_RANK = 500
OVERSAMPLE = 10
ELL = K_RANK + OVERSAMPLE
FP64_PEAK_TFLOPS = 37.1  # profiles/r01_fp64_peak.jsonl: DMMA m8n8k4 microbenchmark, this pool's B200
FP64_PEAK_SOURCE = "profiles/r01_fp64_peak.jsonl (tools/microbench/fp64_peak.cu; MEASURED_PEAKS.json has no FP64 entry)"


def flops_model(m, n, k, ell):
    """Algorithmic FP64 flop counts."""
    cpqr_y = sum(4.0 * (ell - s) * (n - s - 1) for s in range(min(ell, n)))
    cpqr_ct = sum(4.0 * (k - s) * (m - s - 1) for s in range(k))
    return {
        "sketch": 2.0 * ell * m * n,
        "cpqr_y": cpqr_y,
        "t_col": float(k) * k * (n - k),
        "cpqr_ct": cpqr_ct,
        "t_row": float(k) * k * (m - k),
        "qr_c_rt": 2 * 2.0 * k * k * (m + n),
        "cta": 2.0 * k * m * n,
        "ctar": 2.0 * k * k * n,
    }


def cpqr_bytes(rows, cols, steps):
    """Algorithmic HBM bytes of the fused CPQR pass: trailing block read+write
    plus 32 B/column of norm state, per step."""
    return sum(16.0 * (rows - s) * (cols - s) + 32.0 * (cols - s) for s in range(steps))


def ozaki_split_bytes(rows, cols):
    """colmax pass (read) + split pass (read 8 B, write 16 residue bytes) per element."""
    return 32.0 * rows * cols


def measured_traffic(cfg):
    """DRAM bytes per stage launch from the newest committed ncu capture
    (profiles/rNN_traffic.json, C4 shapes only), else None."""
    if (cfg.m, cfg.n, cfg.k) != (M, N, K_RANK):
        return {}
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))  # the newest round's capture
    try:
        with open(files[-1]) as f:
            return json.load(f).get("per_launch", {})
    except Exception:
        return {}


def kernel_rooflines(cfg, st, per_step, engine):
    """Roofline entries of the step's big kernels from their CUDA-event stage
    times (average per launch).  `traffic`: DRAM bytes per launch measured by
    ncu (the newest profiles/rNN_traffic.json) where captured."""
    peaks = read_peaks()
    traffic = measured_traffic(cfg) if engine == "ozaki" else {}
    hbm = peaks.get("hbm_gbs", 6548.5)
    ell = cfg.k + OVERSAMPLE
    out = {}
    if engine == "ozaki":
        i8, i8_src = int8_peak(peaks)
        for name, cols, what in (("sketch_gemm", ell, "Y = Omega A"), ("ctA_gemm", cfg.k, "X^T = A^T Q_c")):
            if st.get(name):
                ops = 16 * 2.0 * cols * cfg.m * cfg.n
                ach = ops / (st[name] * 1e-3) / 1e12
                out[name] = {"kernel": f"imma_gemm_kernel + crt4_kernel ({what}, 16 INT8 residue GEMMs)",
                             "bound": "tensor", "achieved": round(ach, 1), "peak": round(i8, 1), "unit": "TOP/s",
                             "frac": round(ach / i8, 4), "traffic": traffic.get(name),
                             "peak_source": i8_src,
                             "frac_vs_burst": round(ach / int8_burst(), 4) if int8_burst() else None,
                             "algorithmic": f"16 moduli x 2*{cols}*m*n = {ops:.4e} int8 op per launch"}
        if st.get("ozaki_split"):
            # the split stage closes twice per CUR (A + Omega before the sketch, Q_c before
            # A^T Q_c): its per-step total covers every split of the step
            b = (ozaki_split_bytes(cfg.m, cfg.n) + ozaki_split_bytes(cfg.m, ell) + ozaki_split_bytes(cfg.m, cfg.k))
            ach = b / (per_step["ozaki_split"] * 1e-3) / 1e9
            out["ozaki_split"] = {"kernel": "colmax_kernel + split_kernel (A, Omega^T, Q_c residue planes)",
                                  "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                                  "frac": round(ach / hbm, 4), "traffic": traffic.get("ozaki_split"),
                                  "algorithmic": "32 B per element of each split operand (read 8 + 8, write 16)"}
    else:
        for name, key, what in (("sketch_gemm", "sketch", "Y = Omega A"), ("ctA_gemm", "cta", "X^T = A^T Q_c")):
            if st.get(name):
                fm = flops_model(cfg.m, cfg.n, cfg.k, ell)
                ach = fm[key] / (st[name] * 1e-3) / 1e12
                out[name] = {"kernel": f"gemm_tn_kernel ({what}, FP64 DMMA)", "bound": "tensor",
                             "achieved": round(ach, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                             "frac": round(ach / FP64_PEAK_TFLOPS, 4), "traffic": None,
                             "peak_source": FP64_PEAK_SOURCE, "algorithmic": f"{fm[key]:.4e} flop per launch"}
    for name, rows, cols, steps in (("cpqr_sample", ell, cfg.n, ell), ("cpqr_ct", cfg.k, cfg.m, cfg.k)):
        if st.get(name):
            b = cpqr_bytes(rows, cols, steps)
            ach = b / (st[name] * 1e-3) / 1e9
            tb = traffic.get(name)
            meas = tb / (st[name] * 1e-3) / 1e9 if tb else None
            kern = ("cpqr_lazy_kernel x32 + panel_finalize_kernel x32 (bound-pruned panel CPQR: per step only the "
                    "columns whose norm bound can reach the maximum are caught up; one cooperative launch per 16 "
                    "steps, DMMA end-of-panel catch-up + rank-16 update, logical column swaps)") if cols >= 32768 else (
                    "cpqr_panel_kernel x16 + panel_update_dmma_kernel x15 (delayed-update CPQR, one cooperative "
                    "launch per 32 steps, logical column swaps)")
            out[name] = {"kernel": kern,
                         "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(ach / hbm, 4), "traffic": tb,
                         "measured_bytes_gbs": round(meas, 1) if meas else None,
                         "measured_bytes_frac": round(meas / hbm, 4) if meas else None,
                         "measured_bytes_note": "ncu DRAM bytes of the panel form (traffic) / this stage's time: "
                                                "the fraction of HBM the kernel actually moves; `frac` divides the "
                                                "right-looking algorithmic count (SURVEY 8d), which the panel form "
                                                "does not move",
                         "algorithmic": f"SURVEY 8d right-looking count sum_s 16 (rows-s)(cols-s) + 32 (cols-s) "
                                        f"= {b:.4e} B per launch (the panel form moves less: see traffic)",
                         "note": "latency-bound per step (candidate loads -> catch-up -> CTA argmax -> grid "
                                 "barrier -> reflector staging); runs at the power-capped SM clock left by the INT8 "
                                 "GEMMs; tools/bench_cpqr.py with LRB_CPQR_TRACE=1 breaks it down"}
    return out


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


INT8_PEAK_FILE = os.path.join(ROOT, "profiles", "r02_int8_peak.json")


def int8_burst():
    try:
        with open(INT8_PEAK_FILE) as f:
            return float(json.load(f)["int8_tops"])
    except Exception:
        return None


def int8_peak(peaks):
    """Dense INT8 tensor peak (TOP/s) for a kernel timed inside the long,
    power-capped step: the sustained cuBLASLt IMMA figure measured on this
    pool's B200 by tools/microbench/int8_peak.py (committed under profiles/),
    else 2 x the driver's sustained bf16 figure (the B200 INT8 rate is 2x bf16)."""
    try:
        with open(INT8_PEAK_FILE) as f:
            rec = json.load(f)
        return float(rec["int8_tops_sustained"]), (
            "profiles/r02_int8_peak.json: torch._int_mm (cuBLASLt IMMA) 8192^3 back to back, sustained "
            f"(burst {rec.get('int8_tops')} TOP/s)")
    except Exception:
        return 2.0 * peaks.get("bf16_tflops_sustained", 1393.6), \
            "2 x bf16_tflops_sustained of MEASURED_PEAKS.json (INT8 = 2x bf16 rate; no measured INT8 file)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region through
    NVML in a background thread (an `nvidia-smi -lms` subprocess was measured
    to slow the library's launches down by up to 2x on this driver; NVML
    queries at 200 ms do not).  Falls back to nvidia-smi when NVML is absent."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index, period=0.1):
        self.index = index
        self.period = period
        self.samples = []
        self.mx = None
        self._stop = threading.Event()
        self.thread = None

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def run():
                while not self._stop.is_set():
                    try:
                        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(clk), int(rs)))
                    except Exception:
                        pass
                    self._stop.wait(self.period)
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        sm = [c for c, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.mx, "reasons": reasons,
                "samples": len(sm), "source": "NVML (nvmlDeviceGetClockInfo / GetCurrentClocksEventReasons)"}


# ------------------------------------------------------------------ CPU reference arm
def cpu_reference_estimate(sample=2048, threads=0, repeats=1):
    """The reference algorithm on the host (oracle port), stage by stage, on a
    C4-shaped sample (sample x sample, width 1024 -> min(sample,1024), k=500,
    p=10) and extrapolated to 65536^2 by each stage's exact size scaling:
    GEMM-like stages by (M/m)(N/n), n-linear stages by N/n, m-linear by M/m.
    Returns (estimated seconds, details)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle
    from paper_1412_8447_b200 import inputs
    o = Oracle()
    o.set_threads(threads)
    cfg = inputs.scaled(inputs.CONFIGS["c4"], sample, sample, width=min(1024, sample), k=K_RANK)
    a = inputs.synthetic_np(cfg)
    m = n = sample
    k, ell = K_RANK, ELL
    t = {}

    def timed(name, fn):
        t0 = time.perf_counter()
        r = fn()
        t[name] = time.perf_counter() - t0
        return r

    for _ in range(repeats):
        y = timed("sketch", lambda: o.sketch_gaussian(a, ell, 1))
        q = timed("cpqr_y", lambda: o.cpqr(y, ell, want_q=True))  # cpqr_full computes q (cpqr.hpp:91-103)
        piv = q["pivots"]
        s1 = q["s"][:k]
        coeff = timed("t_col", lambda: o.coeff_solve(s1[:, :k], s1[:, k:]))
        c = np.asfortranarray(a[:, piv[:k]])
        rp, rc, sk = timed("tsid", lambda: o.tsid(a, k, piv))
        r = np.asfortranarray(a[rp[:k], :])
        rpinv = timed("pinv_r", lambda: o.pinv(r))
        cpinv = timed("pinv_c", lambda: o.pinv(c))
        x = np.empty((k, n), order="F")
        timed("cpinv_a", lambda: o.L.lro_gemm_nn(k, n, m, cpinv.ctypes.data, k, a.ctypes.data, m, x.ctypes.data, k))
        u = np.empty((k, k), order="F")
        timed("x_rpinv", lambda: o.L.lro_gemm_nn(k, k, n, x.ctypes.data, k, rpinv.ctypes.data, n, u.ctypes.data, k))
    fm, fn_ = M / m, N / n
    scale = {"sketch": fm * fn_, "cpqr_y": fn_, "t_col": fn_, "tsid": fm, "pinv_r": fn_, "pinv_c": fm,
             "cpinv_a": fm * fn_, "x_rpinv": fn_}
    # the reference's cur-pinv path computes pinv(r) twice: once inside
    # cur_from_two_sided (cur.hpp:30) and again in lowrank_main.cpp:215
    mult = {"pinv_r": 2.0}
    est = sum(t[s] * scale[s] * mult.get(s, 1.0) for s in t)
    sample_secs = sum(t.values()) + t["pinv_r"]
    return est, {"stage_seconds_sample": {s: round(v, 4) for s, v in t.items()}, "sample_seconds": sample_secs,
                 "scale": scale, "sample": f"{m}x{n} C4-shaped (width {cfg.width}), k={k}, p={OVERSAMPLE}"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_c4(cfg):
    """The C4 matrix in host memory: built on the GPU with plain torch when one
    is present (inputs.synthetic_torch: no product kernels involved), else
    with numpy.  Input plumbing, untimed."""
    from paper_1412_8447_b200 import inputs
    try:
        import torch
        if torch.cuda.is_available():
            a_dev = inputs.synthetic_torch(cfg, device="cuda", col_block=8192)
            host = np.empty((cfg.m, cfg.n), order="F")
            ht = torch.from_numpy(host)
            for j0 in range(0, cfg.n, 4096):
                ht[:, j0:j0 + 4096].copy_(a_dev[:, j0:j0 + 4096])
            del a_dev, ht
            torch.cuda.empty_cache()
            return host, "GPU (plain torch), copied to host"
    except Exception:
        pass
    return inputs.synthetic_np(cfg), "numpy"


def oracle_workload(o, cfg, a, workload):
    """One full CPU run of a BASELINE configuration on the oracle; returns
    (stage seconds, outputs).  C4 goes stage by stage (tools/c4_full_oracle.py)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    if workload == "c4":
        from c4_full_oracle import run_oracle_cur
        out, t = run_oracle_cur(o, a, cfg.k, cfg.oversample, cfg.sketch_seed, log=lambda *_: None)
        return t, out
    t0 = time.perf_counter()
    if workload == "c1":
        piv, coeff = o.id_column(a, cfg.k)
        out = dict(col_pivots=piv, col_coeff=coeff)
    elif workload == "c2":
        out = o.cur_id(a, cfg.k, u_mode=1)
    else:
        piv, coeff = o.randomized_id(a, cfg.k, cfg.oversample, cfg.sketch_seed)
        out = dict(col_pivots=piv, col_coeff=coeff)
    return {"total": time.perf_counter() - t0}, out


WORKLOAD_TEXT = {
    "c1": "deterministic column ID, BASELINE configs[0] (1000x800, s_j = e^-j/20, k=50)",
    "c2": "deterministic CUR, BASELINE configs[1] (4000x3000, s_j = (j+1)^-2, k=100, U = C^+ A R^+)",
    "c3": "randomized column ID, BASELINE configs[2] (20000^2, width 2000, s_j = e^-j/40, k=200, p=10)",
    "c4": "randomized CUR + tsID, BASELINE configs[3] (65536^2, width 1024, k=500, p=10, U = C^+ A R^+)",
}
METRIC = {
    "c1": "time-to-ID (s), deterministic column ID 1000x800 k=50",
    "c2": "time-to-CUR (s), deterministic CUR 4000x3000 k=100",
    "c3": "time-to-ID (s), randomized column ID 20000^2 k=200",
    "c4": "time-to-CUR (s), randomized CUR 65536^2 k=500",
}


def run_reference(args, rank, world):
    """The reference's CPU path (oracle port) on this host, at the FULL
    configuration.  C4 runs once (minutes); C1-C3 five times (median).  Only
    rank 0 works under torchrun."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle
    from paper_1412_8447_b200 import inputs
    wl = args.workload if args.workload in ("c1", "c2", "c3") else "c4"
    cfg = inputs.CONFIGS[wl]
    threads = os.cpu_count() or 1
    o = Oracle()
    o.set_threads(threads)
    t0 = time.time()
    if wl == "c4":
        a, where = host_c4(cfg)
    else:
        a, where = inputs.synthetic_np(cfg), "numpy"
    gen_s = time.time() - t0
    runs = 1 if wl == "c4" else 5
    totals, stages, out = [], None, None
    for _ in range(runs):
        t0 = time.perf_counter()
        stages, out = oracle_workload(o, cfg, a, wl)
        totals.append(time.perf_counter() - t0)
    value = float(np.median(totals))
    det = {"stage_seconds": {s_: round(v, 3) for s_, v in stages.items()}, "run_seconds": [round(v, 3) for v in totals],
           "cpu_model": cpu_model(), "nproc": os.cpu_count(), "threads": threads, "input": where,
           "input_gen_s": round(gen_s, 1), "requested": {"steps": args.steps, "warmup": args.warmup}}
    if wl == "c4":
        from paper_1412_8447_b200 import inputs as _in
        gold = os.path.join(ROOT, "tests", "golden", "c4_full.npz")
        if os.path.exists(gold):
            g = np.load(gold)
            same_input = str(g["a_sha256"]) == _in.sha256_colblocks(a)
            det["golden_check"] = {"same_input_sha256": same_input,
                                   "col_pivots_equal": bool(np.array_equal(out["col_pivots"], g["col_pivots"])),
                                   "row_pivots_equal": bool(np.array_equal(out["row_pivots"], g["row_pivots"]))}
        # single-thread figure of the sketch (exactly linear in the column count: 1024 of the
        # 65536 columns, x64), the reference's own build being single-threaded Eigen
        o.set_threads(1)
        t0 = time.perf_counter()
        o.sketch_gaussian(np.asfortranarray(a[:, :1024]), cfg.k + cfg.oversample, cfg.sketch_seed)
        ts = time.perf_counter() - t0
        o.set_threads(threads)
        det["single_thread_sketch_s"] = round(ts * cfg.n / 1024, 1)
    line = {
        "metric": METRIC[wl],
        "impl": "reference",
        "value": value,
        "unit": "s",
        "n_gpus": args.gpus,
        "steps": runs,
        "warmup": 0,
        "ms_per_step": value * 1e3,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded U diag(s) V^T, BASELINE spectrum)",
        "config": {"workload": WORKLOAD_TEXT[wl], "m": cfg.m, "n": cfg.n, "k": cfg.k,
                   "oversample": cfg.oversample, "u_mode": "cpinv_a_rpinv" if wl in ("c2", "c4") else None},
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": "port",
                         "sample": f"the full {cfg.m}x{cfg.n} configuration, no sampling ("
                                   f"{'one run' if runs == 1 else 'median of 5 runs'}); oracle/lowrank_oracle.c on "
                                   f"{threads} threads of {cpu_model()}"},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "details": det,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1412_8447_b200 as lr
    from paper_1412_8447_b200 import inputs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = inputs.CONFIGS["c4"]
    cfg = inputs.Config(cfg.name, args.m, args.n, min(cfg.width, args.m, args.n), cfg.spectrum, args.k,
                        OVERSAMPLE, cfg.pipeline, cfg.seed + rank, cfg.sketch_seed)
    ctx = lr.Context(local_rank)
    lr.lowrank._default = ctx
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8 if args.engine == "ozaki" else ctx.GEMM_DMMA)

    t0 = time.time()
    a = inputs.synthetic_torch(cfg, device=dev, col_block=8192)
    gen_s = time.time() - t0
    sk = lr.SketchConfig(oversample=OVERSAMPLE, seed=cfg.sketch_seed, power=args.power)
    out = None
    for _ in range(args.warmup):
        out = lr.randomized_cur_device(a, cfg.k, sk, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx, out=out)
    torch.cuda.synchronize()
    ctx.reset_stats()
    ctx.enable_timing(True)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    launches0 = ctx.kernel_launches()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            out = lr.randomized_cur_device(a, cfg.k, sk, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx, out=out)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = ctx.kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    stages = ctx.stage_report()
    ctx.enable_timing(False)
    stats = ctx.stats()
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # The timed steps ran the CUR's tail as two concurrent chains (row ID of C
    # next to A^T Q_c, lr_ctx_set_concurrent_tail): their stage marks lump the
    # chains together.  A few extra untimed-for-the-metric steps with the
    # sequential tail give the per-kernel times the secondary rooflines need.
    seq_stages, seq_steps, seq_ms = None, 0, None
    if stats.get("concurrent_tail") and not args.no_seq_profile:
        seq_steps = max(1, min(3, args.steps))
        ctx.set_concurrent_tail(0)
        out = lr.randomized_cur_device(a, cfg.k, sk, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx, out=out)
        torch.cuda.synchronize()
        ctx.reset_stats()
        ctx.enable_timing(True)
        ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2.record(stream)
        for _ in range(seq_steps):
            out = lr.randomized_cur_device(a, cfg.k, sk, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx, out=out)
        ev3.record(stream)
        torch.cuda.synchronize()
        seq_ms = ev2.elapsed_time(ev3) / seq_steps
        seq_stages = ctx.stage_report()
        ctx.enable_timing(False)
        ctx.set_concurrent_tail(-1)

    # accuracy (outside the timed region): ||A - CUR||_F / ||A||_F
    err, na = lr.cur_error_fro_device(a, out, ctx=ctx)

    # e2e through the host C ABI: pinned host A, factors copied back
    e2e = None
    if not args.no_e2e:
        host = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True).T
        host.copy_(a)
        del a
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        ha = host.numpy()
        e2e_steps = args.e2e_steps or args.steps
        hout = lr.pinned_cur_outputs(cfg.m, cfg.n, cfg.k)  # reused page-locked result buffers
        for _ in range(2):  # warm-up (the first calls grow the arena and the pinned staging)
            cur = lr.randomized_cur(ha, cfg.k, sk, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx, out=hout)
        barrier()
        e2e_timing = os.environ.get("BENCH_E2E_TIMING") is not None  # diagnostic: stage marks in the e2e calls
        if e2e_timing:
            ctx.reset_stats()
            ctx.enable_timing(True)
        t0 = time.perf_counter()
        step_s = []
        for _ in range(e2e_steps):
            ts = time.perf_counter()
            cur = lr.randomized_cur(ha, cfg.k, sk, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx, out=hout)
            step_s.append(round(time.perf_counter() - ts, 4))
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        if e2e_timing:
            print(json.dumps({"e2e_stages": ctx.stage_report()}), file=sys.stderr)
            ctx.enable_timing(False)
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        k = cfg.k
        d2h = 8 * (cfg.n + cfg.m) + 8 * (cfg.m * k + k * k + k * cfg.n + k * (cfg.n - k) + k * (cfg.m - k) + k * k)
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": 8 * cfg.m * cfg.n, "d2h_bytes_per_step": d2h,
               "steps": e2e_steps, "step_s": step_s, "host_buffer": "pinned A and pinned result buffers",
               "pipeline": "A uploaded in column chunks on a copy stream, each chunk sketched as it lands; "
                           "finished factors copied back on a second stream during the rest of the CUR"}

    if rank != 0:
        return
    fm = flops_model(cfg.m, cfg.n, cfg.k, cfg.k + OVERSAMPLE)
    total_flops = sum(fm.values())
    st = {k: v["ms"] / max(1, v["count"]) for k, v in stages.items()}
    per_step = {k: v["ms"] / args.steps for k, v in stages.items()}
    st_k, per_step_k = dict(st), dict(per_step)
    if seq_stages:  # stages the concurrent tail lumps together: from the sequential profile steps
        for k_, v in seq_stages.items():
            if k_ not in st_k:
                st_k[k_] = v["ms"] / max(1, v["count"])
                per_step_k[k_] = v["ms"] / seq_steps
    kern = kernel_rooflines(cfg, st_k, per_step_k, args.engine)
    # the headline roofline is the dominant kernel: the single stage launch with
    # the longest duration (the ozaki_split entry sums several split launches
    # of different operands, so its per-step share is not one kernel's)
    dom = max(kern, key=lambda n: st.get(n, 0.0)) if kern else None
    def share(n):
        if n in per_step:
            return {"share_of_step": round(per_step[n] / ms, 4)}
        return {"share_of_step": None, "share_of_sequential_step": round(per_step_k.get(n, 0.0) / seq_ms, 4),
                "timed_in": "sequential-tail profile steps (this kernel overlaps the other chain in the timed steps)"}
    roof = dict(kern[dom], **share(dom)) if dom else None
    secondary = {n: dict(v, **share(n)) for n, v in kern.items() if n != dom}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        est, det = cpu_reference_estimate(args.cpu_sample, os.cpu_count() or 1)
        cpu = {"value": est, "unit": "s", "cores": os.cpu_count(), "kind": "port",
               "sample": det["sample"] + "; stage times extrapolated to 65536^2 (bounded sample, this run)",
               "details": det}
        try:  # the full-size CPU run of the same configuration (tools/c4_full_oracle.py on a GPU box)
            with open(os.path.join(ROOT, "profiles", "r02_c4_full_cpu.json")) as f:
                full = json.load(f)
            cpu["measured_full_size"] = {"value": full["total_seconds"], "unit": "s", "cores": full["threads"],
                                         "cpu_model": full["cpu_model"], "stage_seconds": full["stage_seconds"],
                                         "source": "profiles/r02_c4_full_cpu.json (one full 65536^2 oracle run; "
                                                   "bench.py --impl reference repeats it)"}
        except Exception:
            pass
    line = {
        "metric": "time-to-CUR (s), randomized CUR 65536^2 k=500",
        "value": ms / 1e3,
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded U diag(s) V^T, C4 spectrum, generated on device)",
        "config": {"workload": "randomized CUR + tsID, BASELINE configs[3] (65536^2, width 1024, k=500, p=10, "
                               "U = C^+ A R^+)", "m": cfg.m, "n": cfg.n, "k": cfg.k, "oversample": OVERSAMPLE,
                   "u_mode": "cpinv_a_rpinv", "l2": "A (34.4 GB) exceeds L2; no flush needed",
                   "power": args.power,
                   "gemm_engine": {"ozaki": "ozaki_int8 (FP64 emulated on INT8 tcgen05, 16 moduli)",
                                   "dmma": "fp64_dmma"}[args.engine],
                   "parallelism": "replicas" if world > 1 else "single"},
        "fp64_tflops": round(total_flops / (ms * 1e-3) / 1e12, 3),
        "algorithmic_flops": total_flops,
        "rel_error_fro": err / na,
        "roofline": roof,
        "roofline_secondary": secondary,
        "stages_ms": {k: round(v, 3) for k, v in per_step.items()},
        "stages_note": "per-step totals of the library's CUDA-event stage marks (each interval closes at the named "
                       "mark); they sum to ms_per_step up to the gaps between calls",
        "stages_ms_sum": round(sum(per_step.values()), 3),
        "tail_schedule": ("concurrent: row ID of C (CPQR of C^T, T, gather R) on a 40-SM partition next to "
                          "Q_c and A^T Q_c on the other 108 SMs (stage tsid_ctA_split); "
                          "stages_sequential_ms: the same step with the sequential tail, measured after the "
                          "timed region for the per-kernel table") if seq_stages else "sequential",
        "stages_sequential_ms": ({k_: round(v["ms"] / seq_steps, 3) for k_, v in seq_stages.items()}
                                 if seq_stages else None),
        "sequential_ms_per_step": round(seq_ms, 3) if seq_ms else None,
        "sequential_note": ("the profile steps run right after the timed region (power-capped, warm GPU) and only "
                            "serve the per-kernel table; like for like the sequential tail measures 123.2 ms per "
                            "step against 119.9-120.4 concurrent (profiles/r02_cur_split_sweep.jsonl)")
        if seq_ms else None,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clk.summary(),
        "lib_stats": stats,
        "input_gen_s": round(gen_s, 2),
    }
    print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, local_rank):
    """Column-sharded randomized CUR (lr_randomized_cur_sharded_d over an NCCL
    communicator the library binds, csrc/shard.cu): strong scaling, the whole
    65536^2 problem split over the ranks; both CPQRs sharded (one all-gather of
    pivot candidates per step), no all-gather of the sample."""
    import torch

    import paper_1412_8447_b200 as lr
    from paper_1412_8447_b200 import distributed as D
    from paper_1412_8447_b200 import inputs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    base = inputs.CONFIGS["c4"]
    cfg = inputs.Config(base.name, args.m, args.n, min(base.width, args.m, args.n), base.spectrum, args.k,
                        OVERSAMPLE, base.pipeline, base.seed, base.sketch_seed)
    ctx = lr.Context(local_rank)
    lr.lowrank._default = ctx
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8 if args.engine == "ozaki" else ctx.GEMM_DMMA)
    D.attach_nccl(ctx, world=world, rank=rank)
    off, n_g = D.shard_bounds(cfg.n, world, rank)
    a = inputs.synthetic_torch(cfg, device=dev, col_block=8192, col_range=(off, n_g))
    sk = lr.SketchConfig(oversample=OVERSAMPLE, seed=cfg.sketch_seed)

    def step(out=None):
        return D.randomized_cur_sharded_device(ctx, a, off, cfg.n, cfg.k, sk, out=out)

    res = None
    for _ in range(args.warmup):
        res = step(res)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    launches0 = ctx.kernel_launches()
    ctx.reset_stats()
    ctx.enable_timing(True)
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res = step(res)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = ctx.kernel_launches() - launches0
    stages = ctx.stage_report()
    ctx.enable_timing(False)
    # roofline of this rank's sketch contraction (its column shard)
    shard_cfg = inputs.Config(cfg.name, cfg.m, n_g, cfg.width, cfg.spectrum, cfg.k, OVERSAMPLE, cfg.pipeline)
    st_avg = {kk: v["ms"] / max(1, v["count"]) for kk, v in stages.items()}
    st_step = {kk: v["ms"] / args.steps for kk, v in stages.items()}
    roof = kernel_rooflines(shard_cfg, st_avg, st_step, args.engine).get("sketch_gemm")
    if roof:
        roof = dict(roof, note=f"rank 0's column shard ({n_g} of {cfg.n} columns)")
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # e2e: each step copies the rank's column shard from pinned host memory
    # into the device buffer, runs the sharded CUR and reads the replicated
    # factors (and the rank's R block) back into pinned host buffers
    e2e = None
    if not args.no_e2e:
        host = torch.empty((n_g, cfg.m), dtype=torch.float64, pin_memory=True).T
        host.copy_(a)
        torch.cuda.synchronize()
        del a, res
        torch.cuda.empty_cache()
        host_np = host.numpy()  # column-major view of the pinned shard

        def pinned(shape, dtype):
            t = torch.empty(tuple(reversed(shape)), dtype=dtype, pin_memory=True)
            return t.numpy().T if len(shape) == 2 else t.numpy()

        k = cfg.k
        hout = {"col_pivots": pinned((cfg.n,), torch.int64), "row_pivots": pinned((cfg.m,), torch.int64),
                "c": pinned((cfg.m, k), torch.float64), "u": pinned((k, k), torch.float64),
                "r_local": pinned((k, n_g), torch.float64), "col_coeff": pinned((k, cfg.n - k), torch.float64),
                "row_coeff": pinned((k, cfg.m - k), torch.float64), "skeleton": pinned((k, k), torch.float64)}
        d2h = sum(v.nbytes for v in hout.values())

        def e2e_step():
            D.randomized_cur_sharded_host(ctx, host_np, off, cfg.n, cfg.k, sk, out=hout)

        e2e_step()  # warm-up
        e2e_steps = args.e2e_steps or args.steps
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": 8 * cfg.m * cfg.n,
               "d2h_bytes_per_step": d2h * world, "steps": e2e_steps,
               "host_buffer": "pinned column shard per rank (1/N of A) and pinned result buffers",
               "pipeline": "lr_randomized_cur_sharded: the shard uploaded in column chunks, each chunk sketched "
                           "as it lands, then the sharded CUR; bytes summed over ranks"}
    stats = ctx.stats()
    D.detach_nccl(ctx)
    if rank != 0:
        return
    fm = flops_model(cfg.m, cfg.n, cfg.k, cfg.k + OVERSAMPLE)
    line = {
        "metric": "time-to-CUR (s), randomized CUR 65536^2 k=500",
        "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded U diag(s) V^T, C4 spectrum, generated on device per column shard)",
        "config": {"workload": "randomized CUR + tsID, BASELINE configs[3], column-sharded", "m": cfg.m,
                   "n": cfg.n, "k": cfg.k, "oversample": OVERSAMPLE, "u_mode": "cpinv_a_rpinv",
                   "parallelism": f"column-sharded x{world} (sharded CPQRs, NCCL)",
                   "l2": "A shard exceeds L2; no flush needed"},
        "fp64_tflops": round(sum(fm.values()) / (ms * 1e-3) / 1e12, 3),
        "gpu_launches": int(launches), "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": None,
        "roofline": roof, "stages_ms": {kk: round(v, 3) for kk, v in st_step.items()}, "lib_stats": stats,
    }
    print(json.dumps(line), flush=True)


def run_config(args, rank, world, local_rank):
    """BASELINE configs[0..2] on one GPU (N > 1: independent replicas), A
    resident in HBM.  C1 (6.4 MB) and C2 (96 MB) fit in the 126 MB L2, so L2
    is flushed (a 256 MB write) before every timed step and each step is timed
    on its own; C3's A (3.2 GB) exceeds L2.  The CPU figure is the oracle's
    full-size run of the same configuration (single thread, the reference's
    own build being single-threaded Eigen; all threads in details)."""
    import torch

    import paper_1412_8447_b200 as lr
    from paper_1412_8447_b200 import inputs

    wl = args.workload
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = inputs.CONFIGS[wl]
    ctx = lr.Context(local_rank)
    lr.lowrank._default = ctx
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_gemm_mode(ctx.GEMM_OZAKI_INT8 if args.engine == "ozaki" else ctx.GEMM_DMMA)
    a_host = inputs.synthetic_np(cfg)
    a = lr.empty_colmajor(cfg.m, cfg.n, dev)
    a.copy_(torch.from_numpy(a_host))
    sk = lr.SketchConfig(oversample=cfg.oversample, seed=cfg.sketch_seed)

    def step(out=None):
        if wl == "c1":
            return lr.id_column_device(a, cfg.k, ctx=ctx, out=out)
        if wl == "c2":
            return lr.cur_id_device(a, cfg.k, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx, out=out)
        return lr.randomized_id_device(a, cfg.k, sk, ctx=ctx, out=out)

    out = None
    for _ in range(args.warmup):
        out = step(out)
    torch.cuda.synchronize()
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev) if wl in ("c1", "c2") else None
    ctx.reset_stats()
    ctx.enable_timing(True)
    launches0 = ctx.kernel_launches()
    times = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            if flush is not None:
                flush.fill_(1.0)  # 256 MB > L2: the step starts cold
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = step(out)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    launches = ctx.kernel_launches() - launches0
    stages = ctx.stage_report()
    ctx.enable_timing(False)
    # millisecond-scale steps: the median is the per-step time (one preempted host
    # sync inside a call would otherwise dominate the mean); the mean is reported too
    ms = float(np.median(times))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    per_step = {kk: v["ms"] / args.steps for kk, v in stages.items()}
    # e2e through the host API (numpy A in, factors out)
    ts = []
    if not args.no_e2e:
        for _ in range(max(1, args.warmup)):
            host_call(lr, wl, a_host, cfg, sk, ctx)
        for _ in range(args.e2e_steps or args.steps):
            t0 = time.perf_counter()
            host_call(lr, wl, a_host, cfg, sk, ctx)
            ts.append(time.perf_counter() - t0)
    if rank != 0:
        return
    roof = None
    ell = cfg.k + cfg.oversample
    if wl == "c3" and per_step.get("sketch_gemm"):
        if args.engine == "ozaki":
            i8, src = int8_peak(read_peaks())
            ops = 16 * 2.0 * ell * cfg.m * cfg.n
            ach = ops / (per_step["sketch_gemm"] * 1e-3) / 1e12
            roof = {"kernel": "imma_gemm_kernel + crt4_kernel (Y = Omega A, 16 INT8 residue GEMMs)", "bound": "tensor",
                    "achieved": round(ach, 1), "peak": i8, "unit": "TOP/s", "frac": round(ach / i8, 4),
                    "traffic": None, "peak_source": src,
                    "algorithmic": f"16 moduli x 2*{ell}*m*n = {ops:.4e} int8 op"}
        else:
            fl = 2.0 * ell * cfg.m * cfg.n
            ach = fl / (per_step["sketch_gemm"] * 1e-3) / 1e12
            roof = {"kernel": "gemm_tn_kernel (Y = Omega A, FP64 DMMA)", "bound": "tensor", "achieved": round(ach, 2),
                    "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": round(ach / FP64_PEAK_TFLOPS, 4),
                    "traffic": None, "peak_source": FP64_PEAK_SOURCE, "algorithmic": f"{fl:.4e} flop"}
    cpu = None
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_lib import Oracle
        o = Oracle()
        res = {}
        for thr in (1, os.cpu_count() or 1):
            o.set_threads(thr)
            vals = []
            for _ in range(3 if wl == "c3" else 5):
                t0 = time.perf_counter()
                oracle_workload(o, cfg, a_host, wl)
                vals.append(time.perf_counter() - t0)
            res[thr] = float(np.median(vals))
        cpu = {"value": res[1], "unit": "s", "cores": 1, "kind": "port",
               "sample": f"the full {cfg.m}x{cfg.n} configuration (median of {3 if wl == 'c3' else 5} runs), "
                         f"single thread of {cpu_model()}",
               "all_threads": {"value": res[os.cpu_count() or 1], "cores": os.cpu_count()}}
    line = {
        "metric": METRIC[wl], "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded U diag(s) V^T, BASELINE spectrum)",
        "config": {"workload": WORKLOAD_TEXT[wl], "m": cfg.m, "n": cfg.n, "k": cfg.k, "oversample": cfg.oversample,
                   "l2": "flushed (256 MB write) before every step" if flush is not None else "A exceeds L2",
                   "gemm_engine": args.engine, "parallelism": "replicas" if world > 1 else "single"},
        "step_ms": [round(t, 4) for t in times],
        "step_ms_mean": round(float(np.mean(times)), 4),
        "value_is": "median of the per-step device times",
        "roofline": roof,
        "stages_ms": {kk: round(v, 4) for kk, v in per_step.items()},
        "e2e": {"value": float(np.mean(ts)), "unit": "s", "h2d_bytes_per_step": 8 * cfg.m * cfg.n,
                "d2h_bytes_per_step": e2e_d2h(wl, cfg), "steps": len(ts),
                "host_buffer": "pageable numpy A and results (host API)"} if ts else None,
        "cpu_baseline": cpu, "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
        "clocks": clk.summary(), "lib_stats": ctx.stats(),
    }
    print(json.dumps(line), flush=True)


def host_call(lr, wl, a_host, cfg, sk, ctx):
    if wl == "c1":
        return lr.id_column(a_host, cfg.k, ctx=ctx)
    if wl == "c2":
        return lr.cur_id(a_host, cfg.k, u_mode=lr.U_CPINV_A_RPINV, ctx=ctx)
    return lr.randomized_id(a_host, cfg.k, sk, ctx=ctx)


def e2e_d2h(wl, cfg):
    m, n, k = cfg.m, cfg.n, cfg.k
    if wl in ("c1", "c3"):
        return 8 * n + 8 * k * (n - k)
    return 8 * (m + n) + 8 * (m * k + k * k + k * n + k * (n - k) + k * (m - k) + k * k)


def run_sparse(args, rank, world, local_rank):
    """BASELINE configs[4]: sparse randomized CUR of a 200000 x 100000 CSR
    matrix with 100 nonzeros per column (k = 300, p = 10).  A secondary line
    (--workload c5); the headline metric is config 4."""
    import torch

    import paper_1412_8447_b200 as lr
    from paper_1412_8447_b200 import inputs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = lr.Context(local_rank)
    lr.lowrank._default = ctx
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    m, n, npc, k = 200000, 100000, 100, 300
    row_ptr, col_idx, val = inputs.synthetic_csr_torch(m, n, npc, seed=1412 + rank, device=dev)
    sk = lr.SketchConfig(oversample=OVERSAMPLE, seed=1)
    res = None
    for _ in range(args.warmup):
        res = lr.randomized_cur_csr_device(row_ptr, col_idx, val, (m, n), k, sk, ctx=ctx)
    torch.cuda.synchronize()
    ctx.reset_stats()
    ctx.enable_timing(True)
    launches0 = ctx.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res = lr.randomized_cur_csr_device(row_ptr, col_idx, val, (m, n), k, sk, ctx=ctx)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    stages = {kk: v["ms"] / max(1, v["count"]) for kk, v in ctx.stage_report().items()}
    ctx.enable_timing(False)
    err, na = lr.cur_error_fro_csr_device(row_ptr, col_idx, val, (m, n), res, ctx=ctx)
    if rank != 0:
        return
    ell = k + OVERSAMPLE
    nnz = int(val.numel())
    spmm_bytes = nnz * (ell * 8 + 16) + n * ell * 8  # one Omega column per nonzero + indices/values + Y
    roof = None
    if stages.get("sketch_spmm"):
        ach = spmm_bytes / (stages["sketch_spmm"] * 1e-3) / 1e9
        hbm = read_peaks().get("hbm_gbs", 6548.5)
        roof = {"kernel": "spmm_csc_kernel (sketch Y = Omega A, sparse A)", "bound": "hbm", "achieved": round(ach, 1),
                "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4), "traffic": None,
                "algorithmic": "nnz * (l*8 + 16) + n*l*8 bytes (one Omega column gathered per nonzero)"}
    line = {
        "metric": "time-to-CUR (s), sparse randomized CUR 200000x100000 (100 nnz/col) k=300",
        "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic CSR (seeded rows, N(0,1)(i+1)^-1/2 (j+1)^-1 values)",
        "config": {"workload": "BASELINE configs[4] sparse randomized CUR", "m": m, "n": n, "nnz": nnz, "k": k,
                   "oversample": OVERSAMPLE, "u_mode": "cpinv_a_rpinv"},
        "rel_error_fro": err / na, "roofline": roof, "stages_ms": {kk: round(v, 3) for kk, v in stages.items()},
        "gpu_launches": int(ctx.kernel_launches() - launches0), "clocks": clk.summary(),
        "cpu_baseline": None, "e2e": None,
        "note": "no reference implementation exists (dense-only reference); parity on densified down-scaled instances",
    }
    print(json.dumps(line), flush=True)


def self_launch(args):
    """--gpus N > 1 without torchrun: re-run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args, rank, world):
    """--dry-run: the multi-rank launch and timing plumbing only (gloo, CPU):
    barrier, max-over-ranks timing, rank 0 prints the line.  No factorization."""
    import torch
    import torch.distributed as dist
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": "launcher self-test", "dry_run": True, "value": float(t.item()), "unit": "s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ranks_seen": world}),
              flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--m", type=int, default=M)
    p.add_argument("--n", type=int, default=N)
    p.add_argument("--k", type=int, default=K_RANK)
    p.add_argument("--cpu-sample", type=int, default=2048)
    p.add_argument("--e2e-steps", type=int, default=0, help="e2e calls timed (0 = --steps)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-seq-profile", action="store_true",
                   help="skip the sequential-tail profile steps after the timed region (ncu launch lists)")
    p.add_argument("--workload", default="c4", choices=["c4", "c1", "c2", "c3", "c5"],
                   help="c4: dense randomized CUR 65536^2 (headline); c1-c3: BASELINE configs[0..2]; "
                        "c5: sparse CSR 200000x100000")
    p.add_argument("--power", type=int, default=0,
                   help="power iterations q (sketch.hpp:148-164; BASELINE configs use q = 0)")
    p.add_argument("--engine", default="ozaki", choices=["ozaki", "dmma"],
                   help="contraction engine of the two A-sized GEMMs (lr_ctx_set_gemm_mode)")
    p.add_argument("--mode", default="auto", choices=["auto", "single", "replicas", "sharded"],
                   help="N>1: 'sharded' (column blocks of A, strong scaling) or 'replicas'")
    p.add_argument("--dry-run", action="store_true", help="launcher self-test on CPU (gloo), no factorization")
    args = p.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        run_dry(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    mode = args.mode if args.mode != "auto" else ("sharded" if world > 1 else "single")
    if args.workload == "c5":
        run_sparse(args, rank, world, local_rank)
    elif args.workload in ("c1", "c2", "c3"):
        run_config(args, rank, world, local_rank)
    elif mode == "sharded":
        run_sharded(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
