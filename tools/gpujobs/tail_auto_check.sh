# does the automatic concurrent tail pay at the smaller end of its range?
o=gpurun_out/t; mkdir -p $o; : > $o/auto.jsonl
for shape in "32768 65536 500" "65536 32768 500" "49152 49152 300"; do
  set -- $shape
  for s in 0 auto 48; do
    echo "{\"m\": $1, \"n\": $2, \"k\": $3, \"tail\": \"$s\"}" >> $o/auto.jsonl
    if [ $s = auto ]; then unset LRB_CUR_SPLIT; else export LRB_CUR_SPLIT=$s; fi
    timeout 400 python bench.py --m $1 --n $2 --k $3 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-seq-profile >> $o/auto.jsonl 2>> $o/auto.err
  done
done
unset LRB_CUR_SPLIT
python - <<'P'
import json
cfg=None
for l in open('gpurun_out/t/auto.jsonl'):
    d=json.loads(l)
    if 'tail' in d: cfg=d; continue
    print(cfg, round(d['ms_per_step'],2), d['lib_stats']['concurrent_tail'])
P
