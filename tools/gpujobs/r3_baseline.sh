# session start check on the restored tree: GPU suite, smoke, C4 line, CPQR trace
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/b0_smi.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout=600 -x > gpurun_out/b0_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b0_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b0_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/b0_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/b0_bench_c4.jsonl 2> gpurun_out/b0_bench_c4.err
LRB_CPQR_TRACE=1 timeout 300 python tools/bench_cpqr.py 510 65536 > gpurun_out/b0_cpqr_trace.log 2>&1
LRB_CPQR_TRACE=1 LRB_CPQR_TRACE_PANELS=1 timeout 300 python tools/bench_cpqr.py 510 65536 > gpurun_out/b0_cpqr_trace_panels.log 2>&1
