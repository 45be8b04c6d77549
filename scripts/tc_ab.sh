#!/bin/bash
# A/B of the tensor-core (tc_fast.cuh) and mma.sync fast paths over the C3 batch sweep.
# Needs an experiments build (RPL_TC_MIN is read only there).  On the GPU box:
#   bash scripts/tc_ab.sh <tag> [sweep]
set -u
TAG=${1:-ab}
SW=${2:-128,512,1024,2048,4096}
OUT=gpurun_out
mkdir -p $OUT
RPL_NVCC_FLAGS=-DRPL_EXPERIMENTS python -m paper_1801_03138_b200.build --force > $OUT/build_$TAG.log 2>&1 || exit 1
for dd in "" "--ddqn"; do
  for tc in 1073741824 0; do
    RPL_TC_MIN=$tc timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --no-gather \
       --sweep $SW $dd > $OUT/ab_${TAG}_tc${tc}${dd}.jsonl 2> $OUT/ab_${TAG}_tc${tc}${dd}.err
    echo "tc=$tc $dd rc=$?"
  done
done
