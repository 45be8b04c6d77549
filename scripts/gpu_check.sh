#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_train.py tests/test_gpu_tcb.py tests/test_gpu_ring_host.py tests/test_gpu_update_size.py tests/test_gpu_distinct.py tests/test_gpu_nccl.py tests/test_gpu_dp_peer.py -x -q > $OUT/pytest52.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest52.txt
python scripts/loss_branch_check.py > $OUT/lbc52.txt 2>&1
timeout 600 python bench.py --no-c5 --no-gather --no-cpu-baseline > $OUT/bench52.json 2> $OUT/bench52.err
timeout 300 python scripts/kernel_times.py --batch 4096 --ddqn > $OUT/kt52_4096.txt 2>&1
