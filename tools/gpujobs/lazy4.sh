o=gpurun_out/lz4
mkdir -p $o
LRB_CPQR_EVENTS=1 LRB_CPQR_TRACE=1 timeout 120 python tools/cmp_lazy.py run /tmp/l_c4.npz 510 65536 c4 > $o/cpqr_c4.jsonl 2> $o/trace_c4.log
LRB_CPQR_EVENTS=1 LRB_CPQR_TRACE=1 timeout 120 python tools/cmp_lazy.py run /tmp/l_g.npz 510 65536 gauss > $o/cpqr_g.jsonl 2> $o/trace_g.log
timeout 600 python -m pytest tests/test_gpu_lazy_cpqr.py -m gpu -q -x -p timeout --timeout=120 --timeout-method=thread > $o/pytest_lazy.log 2>&1; echo "rc=$?" >> $o/pytest_lazy.log
timeout 1200 python -m pytest tests -m gpu -q -p timeout --timeout=300 --timeout-method=thread --durations=15 > $o/pytest_all.log 2>&1; echo "rc=$?" >> $o/pytest_all.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $o/bench.jsonl 2> $o/bench.err; echo "rc=$?" >> $o/bench.err
