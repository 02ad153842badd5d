for mb in 0 40 60 80 100 120; do
  echo "== keep $mb MB" >> gpurun_out/l2keep.log
  LRB_CPQR_L2KEEP=$mb timeout 120 python tools/bench_cpqr.py 510 65536 >> gpurun_out/l2keep.log 2>&1
  LRB_CPQR_L2KEEP=$mb LRB_CPQR_TRACE=1 LRB_CPQR_TRACE_PANELS=1 timeout 120 python tools/bench_cpqr.py 510 65536 2>&1 | grep 't0=' | head -16 >> gpurun_out/l2keep.log
done
