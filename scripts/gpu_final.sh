#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, the default bench line (C2 + embedded C5), the
# C3 Double-DQN sweep in FP32 and BF16, the in-RAM / in-GPU sweep, an ncu launch list of the
# default bench and ncu --set full captures of the top kernels (B = 128 and B = 4096).
set -u
OUT=gpurun_out/final; mkdir -p $OUT
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
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-gather --no-c5 > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fast_" -s 40 -c 4 -o $OUT/ncu_b128 \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-gather --no-c5 > $OUT/ncu_b128.log 2>&1; echo "ncu b128 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tcb_|fast_bwd0" -s 30 -c 6 -o $OUT/ncu_b4096 \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-gather --no-c5 --batch 4096 --ddqn > $OUT/ncu_b4096.log 2>&1; echo "ncu b4096 rc=$?"
