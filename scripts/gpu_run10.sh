#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/t1_trace.py --batch 4096 --ddqn > $OUT/t1trace_4096.txt 2>&1
timeout 300 python scripts/t1_trace.py --batch 1024 --ddqn > $OUT/t1trace_1024.txt 2>&1
timeout 900 python bench.py --steps 2000 --warmup 100 > $OUT/bench10.json 2> $OUT/bench10.err; echo "bench rc=$?"
