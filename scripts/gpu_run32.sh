#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_dp_peer.py -x -q > $OUT/pytest32a.txt 2>&1; echo "dp_peer alone rc=$?"; tail -2 $OUT/pytest32a.txt
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_dp_peer.py -x -q -k "graph_captured or o6" > $OUT/pytest32b.txt 2>&1; echo "pair rc=$?"; tail -2 $OUT/pytest32b.txt
git -C . log -1 --format=%h 2>/dev/null
