# isolate the GPU test that hung in the first round-2 run
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k tie_after_swap > gpurun_out/g2_tie.log 2>&1; echo "tie rc=$?" >> gpurun_out/g2_tie.log
LRB_CPQR_PANEL=0 timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k tie_after_swap > gpurun_out/g2_tie_rl.log 2>&1; echo "tie(right-looking) rc=$?" >> gpurun_out/g2_tie_rl.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solve_edges.py -q -p timeout --timeout=120 > gpurun_out/g2_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/g2_parity.log
timeout 300 python tools/microbench/int8_peak.py --out gpurun_out/r02_int8_peak.json > gpurun_out/g2_int8.log 2>&1; echo "int8 rc=$?" >> gpurun_out/g2_int8.log
