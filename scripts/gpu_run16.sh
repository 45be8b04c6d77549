#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_tcb.py tests/test_gpu_train.py tests/test_gpu_dp_peer.py tests/test_gpu_ring_host.py -x -q > $OUT/pytest16.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest16.txt
for B in 1024 4096; do timeout 300 python scripts/kernel_times.py --batch $B --ddqn > $OUT/kt16_tcb_$B.txt 2>&1; done
timeout 300 python scripts/t1_trace.py --batch 4096 --ddqn > $OUT/t1trace16.txt 2>&1
for dd in "" "--ddqn"; do
  timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --no-e2e --no-gather --no-c5 \
     --sweep 640,1024,2048,4096 $dd > $OUT/sw16${dd}.jsonl 2> $OUT/sw16${dd}.err
done
