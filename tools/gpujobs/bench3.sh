o=gpurun_out/b; mkdir -p $o; : > $o/bench3.jsonl
for i in 1 2 3; do timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-seq-profile >> $o/bench3.jsonl 2>> $o/bench3.err; done
python - <<'P'
import json
for l in open('gpurun_out/b/bench3.jsonl'):
    d=json.loads(l); print(round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['stages_ms']['cpqr_sample'], d['stages_ms']['tsid_ctA_split'], d['stages_ms']['sketch_gemm'], d['stages_ms']['ozaki_split'])
P
