timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -p timeout --timeout=300 -x > gpurun_out/cl_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cl_pytest.log
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cl_bench_c3.jsonl 2> gpurun_out/cl_bench_c3.err
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cl_bench_c2.jsonl 2> gpurun_out/cl_bench_c2.err
