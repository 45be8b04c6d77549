"""Which step graph a loss destination takes (kernel launches per step: +1 with the loss side
branch) and the device / host-enqueue time per step for device and pinned-host destinations,
with and without host-sourced inserts (4 per step, pageable numpy, as bench.py's e2e loop)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03138_b200.binding as b
from inputs import experiences, init_params
cfg = b.DQNConfig(max_batch=128)
rp = b.Replay(100_000, 27, seed=2)
rp.add_many(experiences(100_000, seed=1))
dqn = b.DQN(cfg, init_params(seed=3))
dev = torch.zeros(1, device="cuda")
host = torch.zeros(4096, dtype=torch.float32, pin_memory=True)
pool = experiences(4 * 4096, seed=7)
for adds in (False, True):
    for name, dsts in (("device", [dev] * 4096), ("pinned", [host[i:i + 1] for i in range(4096)]),
                       ("pinned-fixed-slot", [host[0:1]] * 4096)):
        def step(i):
            if adds:
                rp.add(**{k: v[4 * i:4 * i + 4] for k, v in pool.items()})
            dqn.train_step(rp, 128, dsts[i])
        for i in range(50):
            step(i)
        torch.cuda.synchronize()
        l0 = b.kernel_launches()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        s.record()
        for i in range(2000):
            step(i)
        t1 = time.perf_counter()
        e.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"adds={adds} {name}: {(b.kernel_launches() - l0) / 2000:.2f} launches/step, device {s.elapsed_time(e) / 2000 * 1000:.2f} us/step, "
              f"host enqueue {(t1 - t0) / 2000 * 1e6:.2f} us/step, wall {(t2 - t0) / 2000 * 1e6:.2f}")
