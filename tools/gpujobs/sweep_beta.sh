o=gpurun_out/b; mkdir -p $o; : > $o/beta.log
for b in 0 0.85 0.9 0.93 0.95 0.97 0.99; do
  echo "BETA=$b" >> $o/beta.log
  SPECTRUM=c4 LRB_CPQR_BETA=$b LRB_CPQR_TRACE=1 timeout 300 python tools/bench_cpqr.py 510 65536 2>&1 | grep -E "retry|\"ms\"|trace (pass|barrier)" | tail -4 >> $o/beta.log
  echo "BETA=$b gauss" >> $o/beta.log
  LRB_CPQR_BETA=$b LRB_CPQR_TRACE=1 timeout 300 python tools/bench_cpqr.py 510 65536 2>&1 | grep -E "retry|\"ms\"" | tail -2 >> $o/beta.log
done
sed -E 's/"stats": \{[^}]*\}, //' $o/beta.log | cut -c1-170
