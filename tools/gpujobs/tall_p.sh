o=gpurun_out/t; mkdir -p $o; : > $o/tallp.log
for i in 1 2; do for p in 0 40 48 56 64 72; do
  LRB_CUR_SPLIT=$p timeout 400 python bench.py --m 65536 --n 32768 --k 500 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-seq-profile 2>> $o/tallp.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print($p, round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" >> $o/tallp.log
done; done
sort -n $o/tallp.log
