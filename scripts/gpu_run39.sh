#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
RPL_NVCC_FLAGS=-DRPL_EXPERIMENTS python -m paper_1801_03138_b200.build --force > $OUT/build39.log 2>&1 || exit 1
for v in "" "RPL_K2PDL=1" "RPL_K4PDL=1" "RPL_K2PDL=1 RPL_K4PDL=1"; do
  env $v timeout 300 python bench.py --no-c5 --no-gather --no-cpu-baseline --no-e2e --steps 5000 > $OUT/b39.json 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/b39.json').read().strip().splitlines()[-1]);print('$v', round(d['value']), d['ms_per_step']*1000)"
done
