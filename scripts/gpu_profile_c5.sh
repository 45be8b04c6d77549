#!/bin/bash
# Config 5 (84x84x4 u8 states, B = 256) profile pass, one gpurun call: the judged c5 bench line
# (1M ring), then on a 100k ring (same kernels, shorter pre-fill) the ncu launch list, one
# `ncu --set full` capture of one step's kernels, warm CUPTI kernel times and the RPL_TRACE
# phase timeline of the two tensor-core kernels.
# Usage (repo root, on the GPU box):  bash scripts/gpu_profile_c5.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python bench.py --config c5 > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err
echo "c5 bench rc=$?"
CMD="python bench.py --config c5 --capacity 100000 --steps 50 --warmup 5 --no-cpu-baseline --no-gather --no-e2e"
timeout 600 $CMD > $OUT/plain_c5_$TAG.json 2> $OUT/plain_c5_$TAG.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
    --log-file $OUT/launches_c5_$TAG.csv $CMD > $OUT/ncu_launch_c5_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"wide_l0|wide_dw0|wide_reduce|fast_|gather_u8" \
    -s 40 -c 8 -o $OUT/prof_c5_$TAG $CMD > $OUT/ncu_c5_$TAG.log 2>&1
echo "c5 profile rc=$?"
timeout 300 python scripts/c5_profile.py > $OUT/c5_kernel_times_$TAG.txt 2>&1
timeout 300 python scripts/wide_trace.py > $OUT/c5_wide_trace_$TAG.txt 2>&1
echo done
