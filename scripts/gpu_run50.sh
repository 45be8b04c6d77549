#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tcb.py tests/test_gpu_dp_peer.py -x -q > $OUT/pytest50.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest50.txt
for B in 1024 4096; do timeout 300 python scripts/kernel_times.py --batch $B --ddqn > $OUT/kt50_$B.txt 2>&1; done
