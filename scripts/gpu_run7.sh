#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest7.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest7.txt
bash scripts/traffic_capture.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tcb_fwd|tcb_dw1|tcb_l0" -s 30 -c 3 \
  -o $OUT/prof7_tcb4096 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-gather --batch 4096 --ddqn > $OUT/ncu7.log 2>&1
echo "ncu rc=$?"
