timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout=600 -rf > gpurun_out/v1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v1_pytest.log
timeout 300 python tools/bench_cpqr.py 4000 3000 > gpurun_out/v1_tall.log 2>&1
timeout 300 python tools/bench_cpqr.py 1000 800 >> gpurun_out/v1_tall.log 2>&1
for w in c1 c2; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/v1_bench_$w.jsonl 2> gpurun_out/v1_bench_$w.err; done
