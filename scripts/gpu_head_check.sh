#!/bin/bash
# the final HEAD on one B200: the full GPU test tier, smoke, and the default bench line
set -u
OUT=${1:-gpurun_out/head}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --ddqn --sweep 32,128,640,1024,4096 --steps 2000 --warmup 50 --no-e2e --no-gather --no-cpu-baseline > $OUT/sweep_ddqn.jsonl 2> /dev/null; echo "sweep rc=$?"
