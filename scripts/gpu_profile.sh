#!/bin/bash
# One gpurun call: plain bench (the judged line), then the ncu launch list of the same short
# command and one `ncu --set full` capture each of the train-step and gather kernels.
# Usage (from the repo root, on the GPU box):  bash scripts/gpu_profile.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "bench rc=$?"
CMD="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $OUT/plain_$TAG.json 2> $OUT/plain_$TAG.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fast_|train_step" -s 30 -c 4 \
    -o $OUT/prof_train_$TAG $CMD > $OUT/ncu_train_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather -c 2 \
    -o $OUT/prof_gather_$TAG $CMD > $OUT/ncu_gather_$TAG.log 2>&1
echo "profile rc=$?"
