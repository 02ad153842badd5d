timeout 1200 python -m pytest tests/test_gpu_verify.py tests/test_gpu_c4_full.py tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_distributed.py -q -p timeout --timeout=600 --durations=10 -rf -s > gpurun_out/g5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g5_pytest.log
timeout 300 python tools/bench_cpqr.py 4000 3000 > gpurun_out/g5_tall.log 2>&1
timeout 300 python tools/bench_cpqr.py 1000 800 >> gpurun_out/g5_tall.log 2>&1
for w in c1 c2; do timeout 600 python bench.py --workload $w --steps 5 --warmup 2 > gpurun_out/g5_bench_$w.jsonl 2> gpurun_out/g5_bench_$w.err; done
