o=gpurun_out/m; mkdir -p $o; : > $o/p.log
for i in 1 2 3; do for p in 36 40 44 48; do
  LRB_CUR_SPLIT=$p timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-seq-profile 2>> $o/p.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print($p, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['stages_ms']['tsid_ctA_split'])" >> $o/p.log
done; done
sort -n $o/p.log
