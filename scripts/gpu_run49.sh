#!/bin/bash
OUT=gpurun_out
RPL_NVCC_FLAGS=-DRPL_T3A_EPI_TRACE python -m paper_1801_03138_b200.build --force > $OUT/b49.log 2>&1
python scripts/t3a_epi.py 4096 > $OUT/t3aepi.txt 2>&1
python scripts/t3a_epi.py 1024 >> $OUT/t3aepi.txt 2>&1
