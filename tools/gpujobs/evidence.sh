# round-2 evidence on the final build: driver-style bench line, launch list + DRAM traffic of one timed
# CUR, ncu --set full of the top kernels, C1-C3 lines, the reference arm at full size
set -x
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench_c4.jsonl 2> gpurun_out/ev_bench_c4.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:imma_gemm_kernel --launch-skip 6 -c 1 -f -o gpurun_out/ev_imma python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev_ncu_imma.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:split_kernel --launch-skip 3 -c 1 -f -o gpurun_out/ev_split python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev_ncu_split.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cpqr_panel_kernel -c 1 -f -o gpurun_out/ev_panel0 python tools/bench_cpqr.py 510 65536 > gpurun_out/ev_ncu_panel.log 2>&1
for w in c1 c2 c3; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/ev_bench_$w.jsonl 2> gpurun_out/ev_bench_$w.err; done
timeout 600 python bench.py --workload c3 --engine dmma --steps 10 --warmup 3 > gpurun_out/ev_bench_c3_dmma.jsonl 2> gpurun_out/ev_bench_c3_dmma.err
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/ev_bench_c5.jsonl 2> gpurun_out/ev_bench_c5.err
timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev_reference.jsonl 2> gpurun_out/ev_reference.err
