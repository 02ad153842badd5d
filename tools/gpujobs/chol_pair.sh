timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout=600 -rf -x > gpurun_out/cp_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cp_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cp_bench_c4.jsonl 2> gpurun_out/cp_bench_c4.err
