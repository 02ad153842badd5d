"""CPU: the measurement plumbing -- bench.py's roofline entries and headline
choice from synthetic stage reports, and the ncu launch-list tools on a
synthetic CSV (no GPU, no ncu)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bench  # noqa: E402
from paper_1412_8447_b200 import inputs  # noqa: E402


def _cfg():
    base = inputs.CONFIGS["c4"]
    return inputs.Config(base.name, bench.M, bench.N, base.width, base.spectrum, bench.K_RANK, bench.OVERSAMPLE,
                         base.pipeline)


def test_rooflines_from_stage_report():
    stages = {"ozaki_split": {"ms": 28.0, "count": 2}, "sketch_gemm": {"ms": 27.5, "count": 1},
              "cpqr_sample": {"ms": 20.8, "count": 1}, "cpqr_ct": {"ms": 20.1, "count": 1},
              "ctA_gemm": {"ms": 26.1, "count": 1}}
    st = {k: v["ms"] / v["count"] for k, v in stages.items()}
    per_step = {k: v["ms"] for k, v in stages.items()}  # one step
    kern = bench.kernel_rooflines(_cfg(), st, per_step, "ozaki")
    sk = kern["sketch_gemm"]
    ops = 16 * 2.0 * bench.ELL * bench.M * bench.N
    assert abs(sk["achieved"] - round(ops / (27.5e-3) / 1e12, 1)) < 0.2
    assert sk["bound"] == "tensor" and 0 < sk["frac"] < 1.5 and sk["unit"] == "TOP/s"
    assert kern["cpqr_sample"]["bound"] == "hbm" and kern["cpqr_sample"]["unit"] == "GB/s"
    # the split's achieved bandwidth uses its per-step total (both split marks of the step)
    sp = kern["ozaki_split"]
    b = (bench.ozaki_split_bytes(bench.M, bench.N) + bench.ozaki_split_bytes(bench.M, bench.ELL)
         + bench.ozaki_split_bytes(bench.M, bench.K_RANK))
    assert abs(sp["achieved"] - round(b / 28.0e-3 / 1e9, 1)) < 0.2
    if kern["cpqr_sample"]["traffic"]:
        assert kern["cpqr_sample"]["measured_bytes_frac"] < kern["cpqr_sample"]["frac"]
    # the headline is the longest single stage launch: the sketch GEMM, not the
    # split entry that sums the A, Omega and Q_c splits (14 ms per call)
    dom = max(kern, key=lambda n: st.get(n, 0.0))
    assert dom == "sketch_gemm"


def test_cpqr_bytes_and_flops_model():
    assert bench.cpqr_bytes(2, 3, 1) == 16.0 * 2 * 3 + 32.0 * 3
    fm = bench.flops_model(100, 80, 10, 15)
    assert fm["sketch"] == 2.0 * 15 * 100 * 80
    assert fm["cta"] == 2.0 * 10 * 100 * 80


def _write_launch_csv(path, names):
    hdr = ["ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"]
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(hdr)
        for i, (name, ms) in enumerate(names):
            w.writerow([i, name, "gpu__time_duration.sum", "msecond", f"{ms}"])
            w.writerow([i, name, "dram__bytes_read.sum", "Gbyte", "1.0"])
            w.writerow([i, name, "dram__bytes_write.sum", "Gbyte", "0.5"])


def test_launch_step_and_traffic_json(tmp_path, capsys):
    import launch_step
    import traffic_json
    one_cur = [("split_kernel<1>(long)", 18.0), ("imma_gemm_kernel(x)", 26.0), ("crt_kernel(x)", 0.8)]
    one_cur += [("void lrb::cpqr_panel_kernel<0, 8, 0>(PanelArgs)", 1.5), ("panel_update_dmma_kernel(x)", 0.1)] * 2
    one_cur += [("gemm_tn_kernel<0>(x)", 1.0)]
    one_cur += [("void lrb::cpqr_panel_kernel<0, 8, 0>(PanelArgs)", 1.4)] * 2
    one_cur += [("split_kernel<0>(long)", 0.2), ("imma_gemm_kernel(x)", 25.0), ("<unnamed>::crt4_kernel(x)", 0.6)]
    names = one_cur * 4 + [("void gemm_tn_kernel<2>(x)", 170.0)]
    path = tmp_path / "launches.csv"
    _write_launch_csv(path, names)
    launch_step.main(str(path))
    out = capsys.readouterr().out
    assert "imma_gemm_kernel" in out and "total (serialised, cold)" in out
    tot = float(out.strip().splitlines()[-1].split()[-1])
    assert abs(tot - sum(ms for _, ms in one_cur)) < 1e-6  # exactly one CUR
    js = tmp_path / "traffic.json"
    traffic_json.main(str(path), str(js))
    d = json.load(open(js))
    assert d["per_step"]["sketch_gemm"]["launches"] == 2
    assert d["per_step"]["cpqr_sample"]["launches"] == 4 and d["per_step"]["cpqr_ct"]["launches"] == 2
    assert abs(d["per_launch"]["ctA_gemm"] - 2 * 1.5e9) < 1.0
