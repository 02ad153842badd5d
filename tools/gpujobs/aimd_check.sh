o=gpurun_out/b; mkdir -p $o; : > $o/aimd.log
timeout 600 python -m pytest tests/test_gpu_lazy_cpqr.py -x -q 2>&1 | tail -3 >> $o/aimd.log
for sp in c4 gauss; do
  echo "SPECTRUM=$sp adaptive (retry-driven)" >> $o/aimd.log
  SPECTRUM=$sp LRB_CPQR_TRACE=1 timeout 300 python tools/bench_cpqr.py 510 65536 2>&1 | grep -E "retry|\"ms\"|trace (pass|barrier)" | tail -4 >> $o/aimd.log
done
echo "500 x 65536 (C^T-like, c4 spectrum)" >> $o/aimd.log
SPECTRUM=c4 LRB_CPQR_TRACE=1 timeout 300 python tools/bench_cpqr.py 500 65536 2>&1 | grep -E "retry|\"ms\"" | tail -2 >> $o/aimd.log
timeout 400 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-seq-profile > $o/bench_aimd.jsonl 2>> $o/aimd.log
sed -E 's/"stats": \{[^}]*\}, //' $o/aimd.log | cut -c1-170
python -c "
import json;d=json.loads(open('$o/bench_aimd.jsonl').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['stages_ms'])"
