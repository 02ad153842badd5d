o=gpurun_out/lz5
mkdir -p $o
for er in 192 256 128; do
  LRB_CPQR_EAGER_ROWS=$er LRB_CPQR_EVENTS=1 timeout 120 python tools/cmp_lazy.py run /tmp/l_c4.npz 510 65536 c4 >> $o/cpqr.jsonl 2>> $o/ev_$er.log
  LRB_CPQR_EAGER_ROWS=$er LRB_CPQR_EVENTS=1 timeout 120 python tools/cmp_lazy.py run /tmp/l_g.npz 510 65536 gauss >> $o/cpqr.jsonl 2>> $o/ev_$er.log
done
LRB_CPQR_LAZY=0 timeout 120 python tools/cmp_lazy.py run /tmp/e_c4.npz 510 65536 c4 >> $o/cpqr.jsonl 2>&1
timeout 60 python tools/cmp_lazy.py cmp /tmp/l_c4.npz /tmp/e_c4.npz >> $o/cpqr.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_lazy_cpqr.py tests/test_gpu_parity.py -m gpu -q -x -p timeout --timeout=120 --timeout-method=thread > $o/pytest.log 2>&1; echo "rc=$?" >> $o/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $o/bench.jsonl 2> $o/bench.err; echo "rc=$?" >> $o/bench.err
