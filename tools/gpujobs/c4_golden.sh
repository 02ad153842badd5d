nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
lscpu > gpurun_out/g1_lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python tools/c4_full_oracle.py --out gpurun_out --single-thread-probes > gpurun_out/g1_c4_full_oracle.log 2>&1; echo "oracle rc=$?"
cp gpurun_out/c4_full.npz tests/golden/ 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_c4_full.py tests/test_gpu_parity.py -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g1_pytest.log
