"""bench.py plumbing on CPU: `--gpus N` without torchrun re-launches itself
with N ranks (the driver's N > 1 runs must never silently time one rank),
and the reference arm runs the full configuration it names."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_gpus_flag_self_launches_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "0"], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = last_json(p.stdout)
    assert line["n_gpus"] == 2 and line["ranks_seen"] == 2


def test_reference_arm_runs_the_full_c1_configuration():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "c1",
                        "--steps", "20", "--warmup", "5"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = last_json(p.stdout)
    assert line["impl"] == "reference" and line["config"]["m"] == 1000 and line["config"]["n"] == 800
    assert line["steps"] == 5 and line["details"]["requested"] == {"steps": 20, "warmup": 5}
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0
