"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv).  With --last-cur, only the
launches of the last CUR (from the last colmax_kernel of the A split back to
its start) are summed.
    python tools/launch_table.py launches.csv [--json out.json] [--from-kernel NAME --nth-last K]"""
import csv
import json
import sys
from collections import OrderedDict, defaultdict


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and not r[0].startswith("==")]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        d[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        n = r[ki].split("(")[0].replace("lrb::", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        names[int(r[ii])] = n.replace("void ", "")
    return [(i, names[i], d[i]) for i in sorted(d)]


def main():
    path = sys.argv[1]
    out = None
    start_kernel, nth = None, 1
    args = sys.argv[2:]
    while args:
        a = args.pop(0)
        if a == "--json":
            out = args.pop(0)
        elif a == "--from-kernel":
            start_kernel = args.pop(0)
        elif a == "--nth-last":
            nth = int(args.pop(0))
    seq = load(path)
    if start_kernel:
        idx = [k for k, (_, n, _) in enumerate(seq) if start_kernel in n]
        seq = seq[idx[-nth]:] if len(idx) >= nth else seq
    agg = OrderedDict()
    for _, n, m in seq:
        a = agg.setdefault(n, {"launches": 0, "ms": 0.0, "dram_read_gb": 0.0, "dram_write_gb": 0.0})
        a["launches"] += 1
        a["ms"] += m.get("gpu__time_duration.sum", 0.0) / 1e6
        a["dram_read_gb"] += m.get("dram__bytes_read.sum", 0.0) / 1e9
        a["dram_write_gb"] += m.get("dram__bytes_write.sum", 0.0) / 1e9
    print(f"{'kernel':48s} {'n':>5s} {'ms':>9s} {'DRAM rd GB':>11s} {'DRAM wr GB':>11s}")
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
        print(f"{n[:48]:48s} {a['launches']:5d} {a['ms']:9.3f} {a['dram_read_gb']:11.3f} {a['dram_write_gb']:11.3f}")
    if out:
        json.dump(agg, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
