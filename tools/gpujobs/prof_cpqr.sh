# CPQR profiling: per-phase trace at full clock, ncu --set full of an early and a late panel, and the
# right-looking kernel on the C2 shape
LRB_CPQR_TRACE=1 timeout 300 python tools/bench_cpqr.py 510 65536 > gpurun_out/p1_trace.log 2>&1
timeout 300 python tools/bench_cpqr.py 510 65536 > gpurun_out/p1_plain.log 2>&1
timeout 300 python tools/bench_cpqr.py 4000 3000 > gpurun_out/p1_tall.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cpqr_panel_kernel -c 1 -f -o gpurun_out/p1_panel0 python tools/bench_cpqr.py 510 65536 > gpurun_out/p1_ncu0.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cpqr_panel_kernel --launch-skip 14 -c 1 -f -o gpurun_out/p1_panel14 python tools/bench_cpqr.py 510 65536 > gpurun_out/p1_ncu14.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cpqr_kernel -c 1 -f -o gpurun_out/p1_tall python tools/bench_cpqr.py 4000 3000 > gpurun_out/p1_ncutall.log 2>&1
ls -la gpurun_out/
