#!/bin/bash
# T1 variants: epilogue warps x ring slots (kernel times at B = 1024 / 4096 DDQN)
set -u
OUT=gpurun_out; mkdir -p $OUT
for v in "8 4" "16 2" "8 2" "12 2"; do
  set -- $v
  RPL_NVCC_FLAGS="-DRPL_T1_EPW=$1 -DRPL_T1_SLOTS=$2" python -m paper_1801_03138_b200.build --force > $OUT/build14.log 2>&1 || { echo "build $v failed"; tail -3 $OUT/build14.log; continue; }
  timeout 300 python -m pytest tests/test_gpu_tcb.py -x -q -k "tcb_steps" > $OUT/pytest14_$1_$2.txt 2>&1; echo "v=$v pytest rc=$?"
  for B in 1024 4096; do timeout 300 python scripts/kernel_times.py --batch $B --ddqn > $OUT/kt14_$1_$2_$B.txt 2>&1; done
done
