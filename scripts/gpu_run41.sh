#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/dp1_c5_timing.py > $OUT/dp1c5_planes.txt 2>&1
RPL_NVCC_FLAGS=-DRPL_NO_DP_PLANES python -m paper_1801_03138_b200.build --force > $OUT/b41.log 2>&1
timeout 300 python scripts/dp1_c5_timing.py > $OUT/dp1c5_noplanes.txt 2>&1
python - <<'PY' > $OUT/kt41.txt 2>&1
import os, sys, collections
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1801_03138_b200.binding as b
from inputs import experiences_u8, init_params
D = 84 * 84 * 4
cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512, max_batch=256, sync_period=100, lr=1e-4)
rp = b.Replay(4096, D, seed=2, state_dtype="u8")
e = experiences_u8(1024, state_dim=D, seed=1)
for i in range(4): rp.add(**e)
dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=3))
dqn.attach_peers(0, 1, dqn.peer_handle())
loss = torch.zeros(1, device="cuda")
for i in range(20): dqn.train_step(rp, 256, loss)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for i in range(50): dqn.train_step(rp, 256, loss)
    torch.cuda.synchronize()
per = collections.defaultdict(list)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA: per[ev.name[:60]].append(ev.time_range.end - ev.time_range.start)
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])): print(f"{k:60s} n={len(v):4d} mean={np.mean(v):8.2f}")
PY
