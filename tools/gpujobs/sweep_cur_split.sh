# concurrent CUR tail (CPQR(C^T) chain on an SM partition next to A^T Q_c) with the lazy CPQR
out=gpurun_out/s4_cur_split2.jsonl; : > $out
for late in 1 0; do
for s in 32 40 48 56; do
  echo "{\"LRB_CUR_SPLIT\": $s, \"LATE_R\": $late}" >> $out
  LRB_CUR_SPLIT_LATE_R=$late LRB_CUR_SPLIT=$s timeout 400 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline >> $out 2>> gpurun_out/s4_cur_split2.err
done
done
echo '{"LRB_CUR_SPLIT": 0}' >> $out
timeout 400 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline >> $out 2>> gpurun_out/s4_cur_split2.err
python -m pytest tests/test_gpu_split.py -x -q 2>&1 | tail -3 > gpurun_out/s4_split_tests.log
