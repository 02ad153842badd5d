# INT8 power rounds (A's planes as the M-major tcgen05 operand): parity tests, then C4 with q = 1
set -x
o=gpurun_out/p
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q -k "power" -p timeout --timeout=300 2>&1 | tail -25 > $o/tests.log
cat $o/tests.log | tail -15
timeout 600 python bench.py --power 1 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > $o/bench_c4_q1.jsonl 2> $o/bench_c4_q1.err
LRB_POWER_INT8=0 timeout 600 python bench.py --power 1 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $o/bench_c4_q1_dmma_round.jsonl 2> $o/bench_c4_q1_dmma_round.err
tail -c 1500 $o/bench_c4_q1.jsonl; tail -3 $o/bench_c4_q1.err
