o=gpurun_out/b; mkdir -p $o; : > $o/gapmiss.log
for g in 1.9 3 5 8 16; do
  export LRB_CPQR_GAPMISS=$g
  for sp in c4 gauss; do
    echo "GAPMISS=$g SPECTRUM=$sp" >> $o/gapmiss.log
    SPECTRUM=$sp LRB_CPQR_TRACE=1 timeout 300 python tools/bench_cpqr.py 510 65536 2>&1 | grep -E "retry|\"ms\"" | tail -2 | sed -E 's/"stats": \{[^}]*\}, //' | cut -c1-150 >> $o/gapmiss.log
  done
  for i in 1 2; do
  timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-seq-profile 2>> $o/gapmiss.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('bench', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['stages_ms']['cpqr_sample'], d['stages_ms']['tsid_ctA_split'])" >> $o/gapmiss.log
  done
done
cat $o/gapmiss.log
