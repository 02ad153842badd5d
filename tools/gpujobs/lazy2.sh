o=gpurun_out/lz2
mkdir -p $o
for cfg in "510 65536 c4" "510 65536 gauss" "210 20000 c4" "300 5000 zeros" "64 1000 gauss"; do
  set -- $cfg
  tag=$1_$2_$3
  LRB_CPQR_LAZY=0 timeout 120 python tools/cmp_lazy.py run $o/e_$tag.npz $1 $2 $3 >> $o/runs.jsonl 2>> $o/err_e_$tag.log
  LRB_CPQR_TRACE=1 timeout 120 python tools/cmp_lazy.py run $o/l_$tag.npz $1 $2 $3 >> $o/runs.jsonl 2>> $o/err_l_$tag.log
  echo "rc=$?" >> $o/err_l_$tag.log
  timeout 60 python tools/cmp_lazy.py cmp $o/l_$tag.npz $o/e_$tag.npz >> $o/cmp.jsonl 2>&1
done
rm -f $o/*.npz
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -v -x -p timeout --timeout=120 > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
