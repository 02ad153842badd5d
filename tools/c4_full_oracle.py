#!/usr/bin/env python3
"""Full-size BASELINE configs[3] run of the CPU oracle (TEST INFRASTRUCTURE).

Builds the 65536 x 65536 C4 matrix on the GPU with plain torch
(paper_1412_8447_b200/inputs.py: counter-stream Gaussians, QR, matmul -- the
product library is not involved), copies it to host memory, records its
SHA-256 (column-block digest, inputs.sha256_colblocks), and runs the oracle's
restatement of the reference's randomized CUR with U = C^+ A R^+
(sketch.hpp:227-234 then lowrank_main.cpp:215) on all host cores, stage by
stage:

    sketch      Y = Omega A                        sketch.hpp:67-78
    cpqr_y      cpqr_full(Y), l = k + p steps      cpqr.hpp:32-122
    t_col       stabilized_coeff_solve(S11, S12)   solve.hpp:104-145
    tsid        C = A(:,J), id_row(C), skeleton    id.hpp:121-134
    pinv_r      pinv(R) (one-sided Jacobi)         svd.hpp:124-207
    pinv_c      pinv(C)                            svd.hpp:124-207
    cpinv_a     C^+ A                              lowrank_main.cpp:215
    x_rpinv     (C^+ A) R^+                        lowrank_main.cpp:215

Outputs (into --out, default gpurun_out/):
  c4_full.npz   golden fixture: input hash, both index sets, U, the error,
                checksums of both coefficient matrices (Frobenius norm,
                per-column norms, two seeded projections), the oracle's
                norm-recompute counts on Y and C^T;
  c4_full_cpu.json  the measured CPU time of every stage (the `--impl
                reference` arm of bench.py runs the same code).

    python tools/c4_full_oracle.py [--out DIR] [--threads N] [--single-thread-probes]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

PROJ_SEED_G, PROJ_SEED_H = 777, 778


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def coeff_checks(t, prefix):
    """Size-independent checksums of a k x c coefficient matrix: Frobenius
    norm, per-column 2-norms, T g and h^T T for seeded Gaussian g, h."""
    from paper_1412_8447_b200 import inputs
    k, c = t.shape
    g = inputs.gaussian_np(c, 1, PROJ_SEED_G)[:, 0]
    h = inputs.gaussian_np(k, 1, PROJ_SEED_H)[:, 0]
    return {f"{prefix}_fro": np.linalg.norm(t), f"{prefix}_colnorms": np.linalg.norm(t, axis=0),
            f"{prefix}_tg": t @ g, f"{prefix}_ht": h @ t}


def host_c4_matrix(cfg, log):
    """C4 A on the GPU (plain torch), copied to a column-major host array."""
    import torch

    from paper_1412_8447_b200 import inputs
    t0 = time.time()
    a_dev = inputs.synthetic_torch(cfg, device="cuda", col_block=8192)
    log(f"A generated on the GPU in {time.time() - t0:.1f} s")
    t0 = time.time()
    host = np.empty((cfg.m, cfg.n), order="F")
    ht = torch.from_numpy(host)  # same (column-major) strides as a_dev
    step = 4096
    for j0 in range(0, cfg.n, step):
        ht[:, j0:j0 + step].copy_(a_dev[:, j0:j0 + step])
    del a_dev, ht
    torch.cuda.empty_cache()
    log(f"A copied to host in {time.time() - t0:.1f} s")
    return host


def run_oracle_cur(o, a, k, oversample, seed, log=print, checks=True):
    """The reference's randomized CUR + U = C^+ A R^+ on the oracle, stage by
    stage (see the module docstring).  Returns (outputs, stage seconds)."""
    m, n = a.shape
    ell = k + oversample
    t = {}

    def timed(name, fn):
        t0 = time.perf_counter()
        r = fn()
        t[name] = time.perf_counter() - t0
        log(f"  {name:8s} {t[name]:9.2f} s")
        return r

    y = timed("sketch", lambda: o.sketch_gaussian(a, ell, seed))
    q = timed("cpqr_y", lambda: o.cpqr(y, ell, want_q=True))  # cpqr_full computes q (cpqr.hpp:91-103)
    del y
    piv = q["pivots"]
    s1 = np.asfortranarray(q["s"][:k])
    col_coeff = timed("t_col", lambda: o.coeff_solve(s1[:, :k], s1[:, k:]))
    rp, row_coeff, skel = timed("tsid", lambda: o.tsid(a, k, piv))
    c = np.asfortranarray(a[:, piv[:k]])
    r = np.asfortranarray(a[rp[:k], :])
    rpinv = timed("pinv_r", lambda: o.pinv(r))
    cpinv = timed("pinv_c", lambda: o.pinv(c))
    x = np.empty((k, n), order="F")
    timed("cpinv_a", lambda: o.L.lro_gemm_nn(k, n, m, cpinv.ctypes.data, k, a.ctypes.data, m, x.ctypes.data, k))
    u = np.empty((k, k), order="F")
    timed("x_rpinv", lambda: o.L.lro_gemm_nn(k, k, n, x.ctypes.data, k, rpinv.ctypes.data, n, u.ctypes.data, k))
    out = dict(col_pivots=piv, row_pivots=rp, col_coeff=col_coeff, row_coeff=row_coeff, skeleton=skel, c=c, r=r,
               u=u, recomputes_y=q["recomputes"])
    return out, t


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default=os.path.join(ROOT, "gpurun_out"))
    p.add_argument("--threads", type=int, default=0, help="0 = all host cores")
    p.add_argument("--single-thread-probes", action="store_true",
                   help="also time the sketch (on a 1024-column slice) and CPQR(Y) on one thread")
    args = p.parse_args()
    os.makedirs(args.out, exist_ok=True)

    from oracle_lib import Oracle
    from paper_1412_8447_b200 import inputs

    def log(msg):
        print(msg, flush=True)

    cfg = inputs.CONFIGS["c4"]
    k, p_ = cfg.k, cfg.oversample
    a = host_c4_matrix(cfg, log)
    t0 = time.time()
    digest = inputs.sha256_colblocks(a)
    log(f"A sha256 (column blocks of 1024) {digest} in {time.time() - t0:.1f} s")

    o = Oracle()
    threads = args.threads or os.cpu_count() or 1
    o.set_threads(threads)
    log(f"oracle randomized CUR 65536^2 k={k} p={p_}, U = C^+ A R^+, {threads} threads ({cpu_model()})")
    t_all = time.perf_counter()
    out, stages = run_oracle_cur(o, a, k, p_, cfg.sketch_seed, log)
    total = time.perf_counter() - t_all
    log(f"  total    {total:9.2f} s")

    t0 = time.perf_counter()
    err, na = o.cur_error_fro(a, out["c"], out["u"], out["r"])
    t_err = time.perf_counter() - t0
    log(f"rel error {err / na:.16e} ({t_err:.1f} s)")
    t0 = time.perf_counter()
    ct = o.cpqr(np.asfortranarray(out["c"].T), k, want_q=False)
    assert np.array_equal(ct["pivots"][:k], out["row_pivots"][:k])
    log(f"CPQR(C^T) recomputes {ct['recomputes']} ({time.perf_counter() - t0:.1f} s)")

    golden = dict(a_sha256=np.array(digest), m=cfg.m, n=cfg.n, k=k, oversample=p_, seed=cfg.seed,
                  sketch_seed=cfg.sketch_seed, col_pivots=out["col_pivots"], row_pivots=out["row_pivots"],
                  u=out["u"], err=err, na=na, recomputes_y=out["recomputes_y"], recomputes_ct=ct["recomputes"],
                  skeleton=out["skeleton"], proj_seed_g=PROJ_SEED_G, proj_seed_h=PROJ_SEED_H)
    golden.update(coeff_checks(out["col_coeff"], "tcol"))
    golden.update(coeff_checks(out["row_coeff"], "trow"))
    np.savez_compressed(os.path.join(args.out, "c4_full.npz"), **golden)

    rec = {"what": "oracle (C restatement of the reference) randomized CUR, BASELINE configs[3] at full size",
           "m": cfg.m, "n": cfg.n, "k": k, "oversample": p_, "u_mode": "cpinv_a_rpinv",
           "threads": threads, "nproc": os.cpu_count(), "cpu_model": cpu_model(),
           "stage_seconds": {s: round(v, 3) for s, v in stages.items()}, "total_seconds": round(total, 3),
           "error_eval_seconds": round(t_err, 2), "rel_error_fro": err / na, "a_sha256": digest,
           "recomputes_y": out["recomputes_y"], "recomputes_ct": ct["recomputes"]}

    if args.single_thread_probes:
        o.set_threads(1)
        sl = 1024
        t0 = time.perf_counter()
        o.sketch_gaussian(np.asfortranarray(a[:, :sl]), k + p_, cfg.sketch_seed)
        ts = time.perf_counter() - t0
        o.set_threads(threads)
        yfull = o.sketch_gaussian(a, k + p_, cfg.sketch_seed)
        o.set_threads(1)
        t0 = time.perf_counter()
        o.cpqr(yfull, k + p_, want_q=True)
        tc = time.perf_counter() - t0
        o.set_threads(threads)
        rec["single_thread"] = {"sketch_1024_columns_s": round(ts, 3), "sketch_full_s_linear": round(ts * cfg.n / sl, 1),
                                "cpqr_y_s": round(tc, 2),
                                "note": "the sketch is exactly linear in the column count (each column of Y is "
                                        "Omega times one column of A), so 64 x the 1024-column time is the "
                                        "single-thread full-size sketch"}
        log(f"single thread: sketch {ts:.2f} s per 1024 columns (x64 = {ts * 64:.0f} s), CPQR(Y) {tc:.1f} s")
    with open(os.path.join(args.out, "c4_full_cpu.json"), "w") as f:
        json.dump(rec, f, indent=1)
    log(json.dumps(rec))


if __name__ == "__main__":
    main()
