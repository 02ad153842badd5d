# ncu --set full of the M-major INT8 GEMM (Z^T = A Y^T of a power round): 14th imma launch of bench.py --power 1 --steps 1 --warmup 3
o=gpurun_out/n; mkdir -p $o
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:imma_gemm_kernel --launch-skip 13 -c 1 -f -o $o/imma_mn python bench.py --power 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $o/ncu_mn.log 2>&1
python tools/ncu_summary.py $o/imma_mn.ncu-rep > $o/ncu_summary_mn.md 2> $o/ncu_summary_mn.err
ncu -i $o/imma_mn.ncu-rep --page details --csv > $o/imma_mn_details.csv 2>/dev/null
rm -f $o/imma_mn.ncu-rep
cat $o/ncu_summary_mn.md; tail -3 $o/ncu_mn.log | cut -c1-300
timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout=900 2>&1 | tail -3 > $o/pytest_final.log; cat $o/pytest_final.log
