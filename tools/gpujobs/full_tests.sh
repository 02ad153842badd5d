# whole GPU suite (per-test timeout, durations), smoke, short bench lines
timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout=600 --durations=25 -rf > gpurun_out/g3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g3_smoke.log
for w in c1 c2 c3; do timeout 600 python bench.py --workload $w --steps 5 --warmup 2 > gpurun_out/g3_bench_$w.jsonl 2> gpurun_out/g3_bench_$w.err; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/g3_bench_c4.jsonl 2> gpurun_out/g3_bench_c4.err
timeout 600 python bench.py --mode sharded --steps 3 --warmup 2 --no-e2e > gpurun_out/g3_bench_sharded1.jsonl 2> gpurun_out/g3_bench_sharded1.err
