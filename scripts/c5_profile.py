"""Per-kernel device times of the config-5 step (torch.profiler / CUPTI) on a small byte ring."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.argv = ["bench.py", "--config", "c5", "--steps", "30", "--warmup", "3", "--no-cpu-baseline",
            "--no-gather", "--no-e2e", "--capacity", "20000"] + sys.argv[1:]
sys.path.insert(0, ".")
import bench  # noqa: E402

a = bench.parse()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    bench.run_c5(a)
for e in sorted(prof.key_averages(), key=lambda e: -e.device_time_total)[:30]:
    if e.count:
        print(f"{e.key[:60]:60s} n={e.count:4d} mean={e.device_time_total / e.count:8.2f} us")
