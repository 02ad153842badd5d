timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -p timeout --timeout=300 -x > gpurun_out/sp_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sp_pytest.log
for cfg in "0 4" "64 4" "64 2" "32 4" "96 3" "128 3"; do
  set -- $cfg
  LRB_SPLIT_PIPE=$1 LRB_SPLIT_PIPE_CTAS=$2 timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/sp_$1_$2.jsonl 2> gpurun_out/sp_$1_$2.err
done
