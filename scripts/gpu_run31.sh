#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_dp_peer.py tests/test_gpu_train.py -x -q > $OUT/pytest31.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest31.txt
timeout 300 python scripts/dp1_timing.py > $OUT/dp1_31.txt 2>&1
