#!/bin/bash
# a quick GPU check of the large-batch path: parity tests, then per-kernel times and the sweep
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_tcb.py tests/test_gpu_ring_host.py -x -q > $OUT/pytest_chk.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_chk.txt
for B in 1024 4096; do timeout 300 python scripts/kernel_times.py --batch $B --ddqn > $OUT/kt_chk_$B.txt 2>&1; done
timeout 600 python bench.py --ddqn --sweep 640,1024,2048,4096 --steps 1000 --warmup 50 --no-e2e --no-gather --no-cpu-baseline > $OUT/sw_chk.jsonl 2> /dev/null
