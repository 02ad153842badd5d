# (1) finalize-kernel L2 prefetch A/B, (2) lazy CPQR tests, (3) launch list + DRAM bytes of one timed CUR
# (under ncu the automatic tail schedule is sequential)
set -x
o=gpurun_out/f
mkdir -p $o
for pf in 0 1 0 1; do
  echo "LRB_FIN_PREFETCH=$pf" >> $o/fin_prefetch.log
  SPECTRUM=c4 LRB_FIN_PREFETCH=$pf LRB_CPQR_EVENTS=1 timeout 300 python tools/bench_cpqr.py 510 65536 2>&1 | grep -v "whole call" >> $o/fin_prefetch.log
done
timeout 900 python -m pytest tests/test_gpu_lazy_cpqr.py -x -q 2>&1 | tail -3 > $o/lazy_tests.log
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $o/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $o/ncu_launch.log 2>&1
tail -c 300 $o/ncu_launch.log; cat $o/fin_prefetch.log | cut -c1-200; cat $o/lazy_tests.log
