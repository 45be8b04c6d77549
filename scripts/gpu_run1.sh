set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --ddqn --sweep 32,64,128,256,512,1024,2048,4096 --no-e2e --no-gather --no-cpu-baseline --steps 1000 > gpurun_out/sweep_fp32.jsonl 2> gpurun_out/sweep_fp32.err
timeout 600 python bench.py --ddqn --precision bf16 --sweep 32,64,128,256,512,1024,2048,4096 --no-e2e --no-gather --no-cpu-baseline --steps 1000 > gpurun_out/sweep_bf16.jsonl 2> gpurun_out/sweep_bf16.err
tail -3 gpurun_out/*.err
