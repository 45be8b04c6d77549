#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, the default bench line (C2 + embedded C5), the
# C3 Double-DQN sweep in FP32 and BF16, the in-GPU / in-RAM sweeps, one-rank data-parallel
# timings, an ncu launch list of the default bench, ncu --set full captures of the top kernels
# (B = 128, 1024, 4096) and the warm / cold DRAM traffic.   bash scripts/gpu_final.sh [outdir]
set -u
OUT=${1:-gpurun_out/final}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
for pr in fp32 bf16; do
  timeout 900 python bench.py --ddqn --precision $pr --sweep 32,64,128,256,512,640,1024,2048,4096 --steps 2000 --warmup 50 \
    --no-e2e --no-gather --no-cpu-baseline > $OUT/sweep_ddqn_$pr.jsonl 2> $OUT/sweep_ddqn_$pr.err; echo "sweep $pr rc=$?"
done
for ring in device host_batch host; do
  timeout 900 python bench.py --ring $ring --sweep 16,32,64,128,256,1024,4096 --steps 1000 --warmup 50 \
    --no-e2e --no-gather --no-cpu-baseline > $OUT/inram_$ring.jsonl 2> $OUT/inram_$ring.err; echo "inram $ring rc=$?"
done
timeout 900 python bench.py --ring host_batch --distinct --sweep 16,32,64,128,256,1024,4096 --steps 1000 --warmup 50 \
    --no-e2e --no-gather --no-cpu-baseline > $OUT/inram_host_batch_distinct.jsonl 2> $OUT/inram_hbd.err; echo "inram distinct rc=$?"
timeout 300 python scripts/dp1_timing.py > $OUT/dp_one_rank.txt 2>&1
timeout 300 python scripts/dp1_c5_timing.py > $OUT/dp_c5_one_rank.txt 2>&1
timeout 300 python scripts/loss_branch_check.py > $OUT/loss_branch.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-gather --no-c5 > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fast_" -s 40 -c 4 -o $OUT/ncu_b128 \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-gather --no-c5 > $OUT/ncu_b128.log 2>&1; echo "ncu b128 rc=$?"
for B in 1024 4096; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tcb_|fast_bwd0" -s 30 -c 6 -o $OUT/ncu_b$B \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-gather --no-c5 --batch $B --ddqn > $OUT/ncu_b$B.log 2>&1; echo "ncu b$B rc=$?"
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for cc in all none; do
  timeout 600 ncu --cache-control $cc --clock-control none --metrics $M -k regex:"fast_|tcb_" -s 400 -c 40 --csv \
    python bench.py --steps 60 --warmup 10 --no-cpu-baseline --no-e2e --no-gather --no-c5 > $OUT/traffic_b128_$cc.csv 2> /dev/null
  timeout 600 ncu --cache-control $cc --clock-control none --metrics $M -k regex:"fast_|tcb_" -s 120 -c 36 --csv \
    python bench.py --steps 30 --warmup 5 --batch 4096 --ddqn --no-cpu-baseline --no-e2e --no-gather --no-c5 > $OUT/traffic_b4096_$cc.csv 2> /dev/null
done
echo done
