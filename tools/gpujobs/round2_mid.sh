timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout=600 --durations=15 -rf > gpurun_out/g8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g8_pytest.log
timeout 600 python bench.py --mode sharded --steps 2 --warmup 1 > gpurun_out/g8_bench_sharded1.jsonl 2> gpurun_out/g8_bench_sharded1.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/g8_bench_c4.jsonl 2> gpurun_out/g8_bench_c4.err
