cat > /tmp/seed.py <<'PY'
import sys, time, numpy as np, faulthandler
faulthandler.dump_traceback_later(150, exit=True)
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_1412_8447_b200 as lr
from oracle_lib import Oracle
oracle = Oracle()
for seed in [int(x) for x in sys.argv[1:]]:
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(193, 513)); n = int(rng.integers(m // 2 + 1, 4 * m))
    a = oracle.gaussian_matrix(m, n, seed) * (2.0 ** rng.uniform(-4, 4, size=n))[None, :]
    nz = int(rng.integers(0, n // 3))
    if nz: a[:, rng.choice(n, nz, replace=False)] = 0.0
    nd = int(rng.integers(0, n // 5))
    if nd:
        src = rng.choice(n, nd); dst = rng.choice(n, nd); a[:, dst] = -a[:, src]
    rank = int(np.linalg.matrix_rank(a))
    k = int(rng.integers(1, max(2, min(m, rank) + 1)))
    a = np.asfortranarray(a)
    t = time.time(); q = lr.cpqr_partial(a, k); dt = time.time() - t
    o = oracle.cpqr(a, k)
    print(seed, m, n, k, "nz", nz, "nd", nd, "gpu s", round(dt, 3), "pivots equal", bool(np.array_equal(q.pivots, o["pivots"])), flush=True)
PY
o=gpurun_out/lzh
mkdir -p $o
for rep in 1 2 3; do timeout 200 python /tmp/seed.py 0 1 2 3 4 5 6 7 >> $o/seeds.log 2>&1; echo "rc=$?" >> $o/seeds.log; done
timeout 300 python -m pytest tests/test_gpu_c4_full.py -m gpu -q -x -p timeout --timeout=240 --timeout-method=thread -k "vs_oracle" > $o/c4full.log 2>&1; echo "rc=$?" >> $o/c4full.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $o/bench.jsonl 2> $o/bench.err; echo "rc=$?" >> $o/bench.err
