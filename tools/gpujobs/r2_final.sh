# round-2 final evidence (concurrent CUR tail default): whole GPU suite, smoke, drop-in, C4 bench line,
# launch list + DRAM bytes of one timed CUR, ncu --set full of the lazy CPQR kernels, C1-C3/C5 lines
set -x
o=gpurun_out/f
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $o/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout=900 --durations=10 -rf > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench_c4.jsonl 2> $o/bench_c4.err
timeout 600 python bench.py > $o/bench_c4_default.jsonl 2> $o/bench_c4_default.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $o/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-seq-profile > $o/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cpqr_lazy_kernel --launch-skip 2 -c 1 -f -o $o/lazy env SPECTRUM=c4 python tools/bench_cpqr.py 510 65536 > $o/ncu_lazy.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:panel_finalize_kernel --launch-skip 2 -c 1 -f -o $o/fin env SPECTRUM=c4 python tools/bench_cpqr.py 510 65536 > $o/ncu_fin.log 2>&1
python tools/ncu_summary.py $o/lazy.ncu-rep $o/fin.ncu-rep > $o/ncu_summary_lazy.md 2> $o/ncu_summary.err
for r in lazy fin; do
  ncu -i $o/$r.ncu-rep --page details --csv > $o/${r}_details.csv 2>/dev/null
  ncu -i $o/$r.ncu-rep --page source --csv 2>/dev/null | head -c 3000000 > $o/${r}_source.csv
done
rm -f $o/*.ncu-rep
for w in c1 c2 c3 c5; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 > $o/bench_$w.jsonl 2> $o/bench_$w.err; done
du -sh $o; tail -4 $o/pytest.log; tail -2 $o/smoke.log; head -c 400 $o/bench_c4.jsonl
