#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python scripts/dp1_c5_timing.py > $OUT/dp1c5_45a.txt 2>&1
python scripts/c5dp_kernel_times.py > $OUT/kt45a.txt 2>&1
RPL_NVCC_FLAGS=-DRPL_NO_DP_PLANES python -m paper_1801_03138_b200.build --force > $OUT/b45.log 2>&1
python scripts/dp1_c5_timing.py > $OUT/dp1c5_45b.txt 2>&1
python scripts/c5dp_kernel_times.py > $OUT/kt45b.txt 2>&1
