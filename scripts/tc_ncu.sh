#!/bin/bash
# ncu --set full of the tensor-core fast-path kernels at one batch size (experiments build).
#   bash scripts/tc_ncu.sh <tag> <batch> [extra bench args]
set -u
TAG=${1:-tc}; B=${2:-1024}; shift 2
OUT=gpurun_out
mkdir -p $OUT
if [ -z "${NO_BUILD:-}" ]; then
  RPL_NVCC_FLAGS=-DRPL_EXPERIMENTS python -m paper_1801_03138_b200.build --force > $OUT/build_$TAG.log 2>&1 || exit 1
fi
CMD="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-gather --batch $B $*"
RPL_TC_MIN=0 timeout 300 $CMD > $OUT/plain_$TAG.json 2> $OUT/plain_$TAG.err || exit 2
RPL_TC_MIN=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE:-tc_}" -s 10 -c ${NK:-2} \
    -o $OUT/prof_$TAG $CMD > $OUT/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
