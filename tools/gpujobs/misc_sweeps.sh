o=gpurun_out/m; mkdir -p $o; : > $o/misc.log
for lz in 0 1; do
  echo "C3 LRB_CPQR_LAZY=$lz" >> $o/misc.log
  LRB_CPQR_LAZY=$lz timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>> $o/misc.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), d['stages_ms'])" >> $o/misc.log
  for shp in "210 20000" "510 32768" "510 24576" "310 65536"; do
    echo "cpqr $shp LAZY=$lz" >> $o/misc.log
    SPECTRUM=c4 LRB_CPQR_LAZY=$lz timeout 300 python tools/bench_cpqr.py $shp 2>&1 | grep '"ms"' | sed -E 's/"stats": \{[^}]*\}, //' | cut -c1-120 >> $o/misc.log
  done
done
for p in 32 40 48 56; do
  echo "C4 LRB_CUR_SPLIT=$p" >> $o/misc.log
  LRB_CUR_SPLIT=$p timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-seq-profile 2>> $o/misc.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['stages_ms']['tsid_ctA_split'])" >> $o/misc.log
done
cat $o/misc.log
