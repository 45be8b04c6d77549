#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_dp_peer.py tests/test_gpu_u8.py -x -q > $OUT/pytest47.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest47.txt
timeout 300 python scripts/dp1_timing.py > $OUT/dp1_47.txt 2>&1
