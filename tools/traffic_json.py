"""profiles/rNN_traffic.json from an ncu launch list of `bench.py --steps 1
--warmup 3` (metrics gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum): DRAM bytes per stage launch of the timed CUR, the
`traffic` field of bench.py's roofline entries.
    python tools/traffic_json.py launches.csv out.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_step import rows, short  # noqa: E402


def main(path, out):
    ks = rows(path)
    names = [short(k["name"]) for k in ks]
    imma = [i for i, n in enumerate(names) if n.startswith("imma_gemm_kernel")]
    err = [i for i, n in enumerate(names) if n.startswith("gemm_tn_kernel<2>")]
    lo, hi = imma[5] + 1, min(i for i in err if i > imma[7])
    while names[lo].startswith(("crt_kernel", "crt4_kernel")):
        lo += 1
    seg = list(range(lo, hi))

    def tb(ids):
        rd = sum(ks[i].get("dram__bytes_read.sum", 0.0) for i in ids) * 1e9
        wr = sum(ks[i].get("dram__bytes_write.sum", 0.0) for i in ids) * 1e9
        ms = sum(ks[i].get("gpu__time_duration.sum", 0.0) for i in ids)
        return {"launches": len(ids), "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                "ncu_ms": round(ms, 4)}

    cp = [i for i in seg if names[i].startswith(("cpqr_panel_kernel", "cpqr_lazy_kernel", "panel_finalize_kernel",
                                                 "panel_update", "perm_scatter", "move_slots"))]
    # two CPQRs: split at the largest index gap
    gaps = [(cp[j + 1] - cp[j], j) for j in range(len(cp) - 1)]
    cut = max(gaps)[1] + 1
    cpqr_y, cpqr_ct = cp[:cut], cp[cut:]
    im = [i for i in seg if names[i].startswith("imma_gemm_kernel")]
    crt = [i for i in seg if names[i].startswith(("crt_kernel", "crt4_kernel"))]
    split = [i for i in seg if names[i].startswith(("split_kernel", "colmax_kernel"))]
    res = {
        "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control "
                  f"none on `bench.py --steps 1 --warmup 3` ({os.path.basename(path)}), timed CUR only; cold-cache, "
                  f"serialised launches",
        "per_step": {"cpqr_sample": tb(cpqr_y), "cpqr_ct": tb(cpqr_ct), "sketch_gemm": tb([im[0], crt[0]]),
                     "ctA_gemm": tb([im[1], crt[1]]), "ozaki_split": tb(split)},
    }
    res["per_launch"] = {k: v["traffic_bytes"] for k, v in res["per_step"].items()}
    res["per_launch_note"] = ("bytes = dram__bytes_read.sum + dram__bytes_write.sum summed over the launches of one "
                              "stage (CPQR: every panel launch -- eager or bound-pruned -- with its DMMA update / finalize and "
                              "the final permutation; INT8 GEMM: "
                              "imma + crt; split: every colmax + split launch of the step)")
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res["per_step"], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
