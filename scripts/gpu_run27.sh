#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python scripts/loss_branch_check.py > $OUT/lbc27.txt 2>&1
timeout 600 python bench.py --no-c5 --no-gather --no-cpu-baseline > $OUT/bench27.json 2> $OUT/bench27.err; echo "bench rc=$?"
timeout 600 python bench.py --no-c5 --no-gather --no-cpu-baseline --batch 4096 --ddqn --steps 1000 > $OUT/bench27_4096.json 2> $OUT/bench27_4096.err; echo "bench rc=$?"
timeout 300 python scripts/kernel_times.py --batch 4096 --ddqn > $OUT/kt27_4096.txt 2>&1
