#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/t1_trace.py --batch 4096 --ddqn > $OUT/t1trace17.txt 2>&1
timeout 300 python scripts/t1_trace.py --batch 1024 --ddqn > $OUT/t1trace17_1024.txt 2>&1
