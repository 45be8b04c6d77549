#!/bin/bash
# tc_big vs mma.sync crossover + per-kernel times + ncu of the tcb kernels (experiments build)
set -u
OUT=gpurun_out; mkdir -p $OUT
RPL_NVCC_FLAGS=-DRPL_EXPERIMENTS python -m paper_1801_03138_b200.build --force > $OUT/build_x.log 2>&1 || { tail $OUT/build_x.log; exit 1; }
for dd in "" "--ddqn"; do
  for m in 0 1073741824; do
    RPL_TCB_MIN=$m timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --no-e2e --no-gather \
       --sweep 256,384,512,640,768,1024,1536,2048,4096 $dd > $OUT/xo_tcb${m}${dd}.jsonl 2> $OUT/xo_tcb${m}${dd}.err
    echo "tcbmin=$m $dd rc=$?"
  done
done
for B in 1024 4096; do
  timeout 300 python scripts/kernel_times.py --batch $B --ddqn > $OUT/kt_tcb_$B.txt 2>&1
done
RPL_TCB_MIN=1073741824 timeout 300 python scripts/kernel_times.py --batch 1024 --ddqn > $OUT/kt_mma_1024.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tcb_|fast_bwd0" -s 12 -c 6 \
  -o $OUT/prof_tcb4096 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-gather --batch 4096 --ddqn > $OUT/ncu_tcb4096.log 2>&1
echo "ncu rc=$?"
