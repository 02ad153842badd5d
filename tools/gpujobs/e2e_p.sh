o=gpurun_out/e; mkdir -p $o; : > $o/e2e_p.log
for i in 1 2; do for p in 40 48 56; do
  LRB_CUR_SPLIT=$p timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-seq-profile 2>> $o/e2e_p.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print($p, round(d['ms_per_step'],2), round(d['e2e']['value'],4), d['e2e']['step_s'])" >> $o/e2e_p.log
done; done
sort -n $o/e2e_p.log
