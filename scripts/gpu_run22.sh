#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_train.py -k "loss_destination or c1" -x -q > $OUT/pytest22.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest22.txt
timeout 600 python bench.py --no-c5 --no-gather --no-cpu-baseline > $OUT/bench22.json 2> $OUT/bench22.err; echo "bench rc=$?"
timeout 600 python bench.py --no-c5 --no-gather --no-cpu-baseline --batch 4096 --ddqn --steps 1000 > $OUT/bench22_4096.json 2> $OUT/bench22_4096.err; echo "bench rc=$?"
