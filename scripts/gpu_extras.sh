#!/bin/bash
# evidence extras: the default bench 5 times (median of 5 runs) and one ncu --set full
# capture of a config-5 step's kernels
set -u
OUT=${1:-gpurun_out/extras}; mkdir -p $OUT
for r in 1 2 3 4 5; do
  timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_run$r.json 2> /dev/null; echo "bench $r rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wide_|gather_u8|fast_|insert_u8" -s 30 -c 9 \
  -o $OUT/ncu_c5 python bench.py --config c5 --capacity 100000 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-gather > $OUT/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
