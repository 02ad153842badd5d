o=gpurun_out/lz3
mkdir -p $o
for kind in c4 gauss; do
  LRB_CPQR_EVENTS=1 LRB_CPQR_TRACE=1 LRB_CPQR_TRACE_PANELS=1 timeout 120 python tools/cmp_lazy.py run /tmp/l_$kind.npz 510 65536 $kind >> $o/runs.jsonl 2> $o/trace_$kind.log
  LRB_CPQR_EVENTS=1 timeout 120 python tools/cmp_lazy.py run /tmp/l2_$kind.npz 510 65536 $kind >> $o/runs.jsonl 2> $o/events_$kind.log
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cpqr_lazy_kernel --launch-skip 0 -c 1 -f -o /tmp/lazy_p0 python tools/cmp_lazy.py run /tmp/x.npz 510 65536 c4 > $o/ncu_lazy.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:panel_finalize_kernel --launch-skip 0 -c 1 -f -o /tmp/fin_p0 python tools/cmp_lazy.py run /tmp/x.npz 510 65536 c4 > $o/ncu_fin.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p timeout --timeout=300 --timeout-method=thread --durations=20 > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
for r in lazy_p0 fin_p0; do
  ncu -i /tmp/$r.ncu-rep --page details --csv > $o/${r}_details.csv 2>&1
  ncu -i /tmp/$r.ncu-rep --page source --csv > /tmp/${r}_source.csv 2>&1; head -c 3000000 /tmp/${r}_source.csv > $o/${r}_source.csv
done
du -sh $o
