#!/bin/bash
# DRAM bytes per kernel launch of the train step, cold (ncu's default cache flush between
# kernels) and warm (--cache-control none: L2 as the previous kernel left it), at the C2
# headline shape (B = 128 DQN) and the C3 large-batch shape (B = 4096 DDQN).
#   bash scripts/traffic_capture.sh   (on the GPU box; CSVs in gpurun_out/)
set -u
OUT=gpurun_out; mkdir -p $OUT
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for cc in all none; do
  timeout 600 ncu --cache-control $cc --clock-control none --metrics $M -k regex:"fast_|tcb_" -s 400 -c 40 --csv \
    python bench.py --steps 60 --warmup 10 --no-cpu-baseline --no-e2e --no-gather > $OUT/traffic_b128_$cc.csv 2> $OUT/traffic_b128_$cc.err
  timeout 600 ncu --cache-control $cc --clock-control none --metrics $M -k regex:"fast_|tcb_" -s 120 -c 36 --csv \
    python bench.py --steps 30 --warmup 5 --batch 4096 --ddqn --no-cpu-baseline --no-e2e --no-gather > $OUT/traffic_b4096_$cc.csv 2> $OUT/traffic_b4096_$cc.err
done
