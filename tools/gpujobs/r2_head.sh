# round-2 evidence at HEAD (bound-pruned CPQR default): whole GPU suite, smoke, C4 bench line,
# launch list + DRAM bytes of one timed CUR, ncu --set full of the lazy CPQR kernels
set -x
o=gpurun_out/h
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $o/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p timeout --timeout=600 --durations=15 -rf > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench_c4.jsonl 2> $o/bench_c4.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $o/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $o/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cpqr_lazy_kernel --launch-skip 2 -c 1 -f -o $o/lazy env SPECTRUM=c4 python tools/bench_cpqr.py 510 65536 > $o/ncu_lazy.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:panel_finalize_kernel --launch-skip 2 -c 1 -f -o $o/fin env SPECTRUM=c4 python tools/bench_cpqr.py 510 65536 > $o/ncu_fin.log 2>&1
for r in lazy fin; do
  ncu -i $o/$r.ncu-rep --page raw --csv > $o/${r}_raw.csv 2>/dev/null
  ncu -i $o/$r.ncu-rep --page details --csv > $o/${r}_details.csv 2>/dev/null
  ncu -i $o/$r.ncu-rep --page source --csv > $o/${r}_source.csv 2>/dev/null
done
mkdir -p /tmp/keep && mv $o/*.ncu-rep /tmp/keep/ 2>/dev/null
du -sh gpurun_out/* ; ls -la $o
tail -5 $o/pytest.log; tail -3 $o/smoke.log; head -c 600 $o/bench_c4.jsonl; tail -5 $o/bench_c4.err
