for g in 148 128 111 96 74 64; do
  echo "GRID=$g" >> gpurun_out/s4_cpqr_grid.log
  SPECTRUM=c4 LRB_CPQR_GRID=$g LRB_CPQR_TRACE=1 timeout 300 python tools/bench_cpqr.py 510 65536 >> gpurun_out/s4_cpqr_grid.log 2>&1
done
for b in 0.5 0.7 0.9; do
  echo "BETA=$b" >> gpurun_out/s4_cpqr_grid.log
  SPECTRUM=c4 LRB_CPQR_BETA=$b timeout 300 python tools/bench_cpqr.py 510 65536 >> gpurun_out/s4_cpqr_grid.log 2>&1
done
