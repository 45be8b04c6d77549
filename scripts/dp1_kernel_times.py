"""CUPTI kernel times of a one-rank data-parallel learner (B = 128): the peer-memory exchange
attached to itself, and NCCL with a one-rank communicator (RPL_DP_FORCE=1)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RPL_DP_FORCE"] = "1"
import numpy as np, torch
import paper_1801_03138_b200.binding as b
from inputs import experiences, init_params
cfg = b.DQNConfig(max_batch=128)
rp = b.Replay(100_000, 27, seed=2)
rp.add_many(experiences(100_000, seed=1))
for mode in ("p2p", "nccl"):
    dqn = b.DQN(cfg, init_params(seed=3))
    if mode == "p2p":
        dqn.attach_peers(0, 1, dqn.peer_handle())
    else:
        dqn.attach_nccl(0, 1, b.nccl_unique_id())
    loss = torch.zeros(1, device="cuda")
    for i in range(50):
        dqn.train_step(rp, 128, loss)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for i in range(100):
            dqn.train_step(rp, 128, loss)
        torch.cuda.synchronize()
    per = collections.defaultdict(list)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            per[ev.name[:60]].append(ev.time_range.end - ev.time_range.start)
    print(mode)
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k:60s} n={len(v):4d} mean={np.mean(v):7.2f}")
    dqn.close()
