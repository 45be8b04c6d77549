#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python scripts/loss_branch_check.py > $OUT/lbc26.txt 2>&1
timeout 600 python bench.py --no-c5 --no-gather --no-cpu-baseline > $OUT/bench26.json 2> $OUT/bench26.err; echo "bench rc=$?"
timeout 600 python bench.py --no-c5 --no-gather --no-cpu-baseline --batch 4096 --ddqn --steps 1000 > $OUT/bench26_4096.json 2> $OUT/bench26_4096.err; echo "bench rc=$?"
timeout 300 python scripts/kernel_times.py --batch 128 > $OUT/kt26_128.txt 2>&1
timeout 300 python scripts/kernel_times.py --batch 4096 --ddqn > $OUT/kt26_4096.txt 2>&1
