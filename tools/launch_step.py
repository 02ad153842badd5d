"""Per-kernel table of ONE timed C4 CUR from an ncu launch list of
`bench.py --steps 1 --warmup 3` (value path: two imma launches per CUR; the
timed CUR runs from after the 3rd warm-up's ctA contraction to the error GEMM).
    python tools/launch_step.py launches.csv"""
import csv
import sys
from collections import OrderedDict


def rows(path):
    hdr, out = None, {}
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        i = int(d["ID"])
        e = out.setdefault(i, {"name": d["Kernel Name"]})
        v = float(d["Metric Value"].replace(",", "")) if d["Metric Value"] else 0.0
        u = d["Metric Unit"]
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u, 1.0)
        e[d["Metric Name"]] = v * scale
    return [out[i] for i in sorted(out)]


def short(n):
    n = n.split("(")[0].replace("void ", "").replace("lrb::", "").replace("(anonymous namespace)::", "")
    return n.replace("<unnamed>::", "").replace("cpqr_detail::", "")


def main(path):
    ks = rows(path)
    names = [short(k["name"]) for k in ks]
    imma = [i for i, n in enumerate(names) if n.startswith("imma_gemm_kernel")]
    err = [i for i, n in enumerate(names) if n.startswith("gemm_tn_kernel<2>")]
    lo = imma[5] + 1
    hi = min(i for i in err if i > imma[7])
    while lo < hi and names[lo].startswith(("crt_kernel", "crt4_kernel")):
        lo += 1
    tab = OrderedDict()
    for k, n in zip(ks[lo:hi], names[lo:hi]):
        t = tab.setdefault(n, [0, 0.0, 0.0, 0.0])
        t[0] += 1
        t[1] += k.get("gpu__time_duration.sum", 0.0)
        t[2] += k.get("dram__bytes_read.sum", 0.0)
        t[3] += k.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in tab.values())
    print(f"{'kernel':48s} {'n':>4s} {'ms':>9s} {'share':>6s} {'rd GB':>8s} {'wr GB':>8s}")
    for n, (c, ms, rd, wr) in sorted(tab.items(), key=lambda x: -x[1][1]):
        print(f"{n[:48]:48s} {c:4d} {ms:9.3f} {100 * ms / tot:5.1f}% {rd:8.2f} {wr:8.2f}")
    print(f"{'total (serialised, cold)':48s} {sum(v[0] for v in tab.values()):4d} {tot:9.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
