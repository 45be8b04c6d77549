#!/bin/bash
# timing experiment: T1 without its H1 store (results invalid; kernel times only)
set -u
OUT=gpurun_out; mkdir -p $OUT
RPL_NVCC_FLAGS=-DRPL_T1_NOH1 python -m paper_1801_03138_b200.build --force > $OUT/build12.log 2>&1 || exit 1
timeout 300 python scripts/kernel_times.py --batch 4096 --ddqn > $OUT/kt12_noh1_4096.txt 2>&1
RPL_NVCC_FLAGS=-DRPL_T1_NOH1 RPL_TRACE=1 timeout 300 python scripts/t1_trace.py --batch 4096 --ddqn > $OUT/t1trace12.txt 2>&1
