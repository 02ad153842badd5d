# final build: whole GPU suite, smoke, default bench line, 20-step bench line, drop-in suite
set -x
o=gpurun_out/g
mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout=900 --durations=8 -rf > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench_c4.jsonl 2> $o/bench_c4.err
timeout 600 python bench.py > $o/bench_c4_default.jsonl 2> $o/bench_c4_default.err
timeout 600 python bench.py --power 1 --steps 10 --warmup 3 > $o/bench_c4_q1.jsonl 2> $o/bench_c4_q1.err
tail -4 $o/pytest.log; tail -2 $o/smoke.log; head -c 300 $o/bench_c4.jsonl
