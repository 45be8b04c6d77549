#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_train.py tests/test_gpu_tcb.py tests/test_gpu_ring_host.py tests/test_gpu_update_size.py tests/test_gpu_distinct.py tests/test_gpu_dp_peer.py tests/test_gpu_nccl.py tests/test_gpu_u8.py tests/test_gpu_precision.py -x -q > $OUT/pytest25.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest25.txt
timeout 600 python bench.py --no-c5 --no-gather --no-cpu-baseline > $OUT/bench25.json 2> $OUT/bench25.err; echo "bench rc=$?"
timeout 600 python bench.py --no-c5 --no-gather --no-cpu-baseline --batch 4096 --ddqn --steps 1000 > $OUT/bench25_4096.json 2> $OUT/bench25_4096.err; echo "bench rc=$?"
