#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tcb.py -x -q > $OUT/pytest8.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest8.txt
for B in 1024 4096; do timeout 300 python scripts/kernel_times.py --batch $B --ddqn > $OUT/kt8_tcb_$B.txt 2>&1; done
for dd in "" "--ddqn"; do
  timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --no-e2e --no-gather \
     --sweep 640,1024,2048,4096 $dd > $OUT/sw8${dd}.jsonl 2> $OUT/sw8${dd}.err
done
