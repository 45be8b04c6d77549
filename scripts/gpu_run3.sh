#!/bin/bash
# tcb parity + DP/wide tests, then per-kernel times and the tcb / mma.sync crossover
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tcb.py tests/test_gpu_dp_peer.py tests/test_gpu_u8.py -x -q > $OUT/pytest3.txt 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest3.txt
for B in 1024 4096; do timeout 300 python scripts/kernel_times.py --batch $B --ddqn > $OUT/kt3_tcb_$B.txt 2>&1; done
RPL_NVCC_FLAGS=-DRPL_EXPERIMENTS python -m paper_1801_03138_b200.build --force > $OUT/build_x.log 2>&1 || exit 1
for dd in "" "--ddqn"; do for m in 0 1073741824; do
  RPL_TCB_MIN=$m timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --no-e2e --no-gather \
     --sweep 256,384,512,640,768,1024,2048,4096 $dd > $OUT/xo3_tcb${m}${dd}.jsonl 2> $OUT/xo3_tcb${m}${dd}.err
done; done
