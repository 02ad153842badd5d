"""Summarise ncu reports (--set full captures) into one markdown table row per
kernel launch: duration, SM clock, DRAM bytes, throughputs, tensor-pipe
activity, top warp stalls.

    python tools/ncu_summary.py report.ncu-rep [...] > profiles/rNN_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

METRICS = {
    "dur_ms": ("gpu__time_duration.sum", 1.0),
    "sm_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "dram_rd": ("dram__bytes_read.sum", 1.0),
    "dram_wr": ("dram__bytes_write.sum", 1.0),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l2_pct": ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pct": ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fp64_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "occ_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1, "us": 1e-3, "usecond": 1e-3,
              "msecond": 1, "ns": 1e-6, "nsecond": 1e-6, "Ghz": 1, "Mhz": 1e-3, "hz": 1e-9, "%": 1, "": 1}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(head):
            d[h] = (r[i] if i < len(r) else "", units[i] if i < len(units) else "")
        res.append(d)
    return res


def num(d, name):
    for key in (name, "TPC.TriageCompute." + name):
        if key in d:
            v, u = d[key]
            try:
                return float(v.replace(",", "")) * UNIT_SCALE.get(u, 1.0)
            except ValueError:
                return None
    return None


def stalls(d, top=3):
    pre = "smsp__average_warp_latency_issue_stalled_"
    pre2 = "smsp__pcsamp_warps_issue_stalled_"
    vals = []
    for k, (v, _) in d.items():
        if k.startswith(pre2) and k.endswith("") and "not_issued" not in k:
            try:
                vals.append((float(v.replace(",", "")), k[len(pre2):]))
            except ValueError:
                pass
    if not vals:
        for k, (v, _) in d.items():
            if k.startswith(pre) and k.endswith(".ratio"):
                try:
                    vals.append((float(v.replace(",", "")), k[len(pre):-6]))
                except ValueError:
                    pass
    vals.sort(reverse=True)
    return ", ".join(f"{n}" for _, n in vals[:top])


def main():
    print("| report | kernel | ms | SM GHz | DRAM read GB | DRAM write GB | DRAM % | L2 % | SM % | tensor % | "
          "FP64 % | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for rep in sys.argv[1:]:
        for d in raw(rep):
            name = d.get("Kernel Name", ("?", ""))[0].split("(")[0].replace("lrb::", "").replace("<unnamed>::", "")
            name = name.replace("(anonymous namespace)::", "")
            vals = {k: num(d, m) for k, (m, _) in METRICS.items()}

            def f(x, nd=2, s=1.0):
                return "" if x is None else f"{x / s:.{nd}f}"
            print(f"| {rep.split('/')[-1]} | {name} | {f(vals['dur_ms'], 3)} | {f(vals['sm_ghz'])} | "
                  f"{f(vals['dram_rd'], 2, 1e9)} | {f(vals['dram_wr'], 2, 1e9)} | {f(vals['dram_pct'], 1)} | "
                  f"{f(vals['l2_pct'], 1)} | {f(vals['sm_pct'], 1)} | {f(vals['tensor_pct'], 1)} | "
                  f"{f(vals['fp64_pct'], 1)} | {stalls(d)} |")


if __name__ == "__main__":
    main()
