"""Generate tests/golden/golden_small.npz from the REFERENCE's own code.

Runs the unmodified reference headers (/root/reference/proj/include/lowrank)
compiled in place against oracle/eigen_subset (oracle/_ref/liblowrank_ref.so,
`make -C oracle ref`).  Inputs are stored with the outputs so the fixtures
are self-contained on the GPU box (where /root/reference does not exist).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle_lib import Ref  # noqa: E402
from paper_1412_8447_b200 import inputs  # noqa: E402


def main():
    r = Ref()
    out = {}
    # cpqr known cases (test_cpqr.cpp:51-62, :93-115 shapes)
    g = r.gaussian_matrix(10, 8, 7)
    q = r.cpqr(g, 5)
    out.update(cpqr_a=g, cpqr_k=5, cpqr_s=q["s"], cpqr_q=q["q"], cpqr_piv=q["pivots"])
    g = r.gaussian_matrix(15, 11, 3)
    q = r.cpqr(g, 11)
    out.update(cpqrf_a=g, cpqrf_s=q["s"], cpqrf_q=q["q"], cpqrf_piv=q["pivots"])
    # deterministic column ID on a C1-shaped spectrum
    cfg = inputs.scaled(inputs.CONFIGS["c1"], 200, 150, width=150, k=20)
    a = inputs.synthetic_np(cfg)
    p, c = r.id_column(a, 20)
    out.update(id_a=a, id_k=20, id_piv=p, id_coeff=c)
    # randomized ID on a C3-shaped spectrum
    cfg = inputs.scaled(inputs.CONFIGS["c3"], 200, 300, width=150, k=30)
    a = inputs.synthetic_np(cfg)
    p, c = r.randomized_id(a, 30, 10, 5)
    out.update(rid_a=a, rid_k=30, rid_p=10, rid_seed=5, rid_piv=p, rid_coeff=c)
    # randomized CUR on a C4-shaped spectrum, both middle factors
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 200, 240, width=160, k=40)
    a = inputs.synthetic_np(cfg)
    for mode in (0, 1):
        res = r.randomized_cur(a, 40, 10, 7, u_mode=mode)
        for key, val in res.items():
            out[f"rcur{mode}_{key}"] = val
    p, c = r.randomized_id(a, 40, 10, 7)
    rp, rc, sk = r.tsid(a, 40, p, c)
    out.update(rcur_a=a, rcur_k=40, rcur_p=10, rcur_seed=7, rcur_col_coeff=c, rcur_row_coeff=rc, rcur_skeleton=sk)
    # deterministic CUR (C2-shaped spectrum) with u = pinv(C) A pinv(R)
    cfg = inputs.scaled(inputs.CONFIGS["c2"], 160, 120, width=120, k=25)
    a = inputs.synthetic_np(cfg)
    res = r.cur_id(a, 25, u_mode=1)
    out.update(cur_a=a, cur_k=25, **{f"cur_{k}": v for k, v in res.items()})
    path = os.path.join(HERE, "golden_small.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
