"""The bench e2e loop alone on a ring of the given capacity, with host / device / no inserts and
a pinned-host / device loss destination: device, host-enqueue and wall time per step.
    python scripts/e2e_probe.py CAPACITY STEPS"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1801_03138_b200.binding as b
from inputs import experiences, init_params
cfg = b.DQNConfig(state_dim=27, n_actions=8, double_dqn=False, gamma=0.99, lr=1e-4, huber_kappa=1.0,
                  sync_period=10_000, max_batch=128, dueling=True, hidden=(128,), stream=512)
cap = int(sys.argv[1]); K = int(sys.argv[2])
rp = b.Replay(cap, 27, seed=2)
rp.add_many(experiences(cap, seed=1))
dqn = b.DQN(cfg, init_params(seed=3))
pool_h = experiences(1024, seed=7)
pool_d = {k: torch.from_numpy(v).cuda() for k, v in pool_h.items()}
loss_host = torch.zeros(K, dtype=torch.float32, pin_memory=True)
slots = [loss_host[i:i + 1] for i in range(K)]
dev = torch.zeros(1, device="cuda")
for adds in ("host", "device", "none"):
    for dst in ("pinned", "device"):
        def step(i):
            j = (i * 4) % (1024 - 4)
            if adds == "host":
                rp.add(**{kk: v[j:j + 4] for kk, v in pool_h.items()})
            elif adds == "device":
                rp.add(**{kk: v[j:j + 4] for kk, v in pool_d.items()}, defer=True)
            dqn.train_step(rp, 128, slots[i] if dst == "pinned" else dev)
        for i in range(100):
            step(i)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); s.record()
        for i in range(K):
            step(i)
        t1 = time.perf_counter(); e.record(); torch.cuda.synchronize(); t2 = time.perf_counter()
        print(f"cap={cap} adds={adds:6s} loss={dst:7s}: device {s.elapsed_time(e) / K * 1000:.2f} us/step, "
              f"host enqueue {(t1 - t0) / K * 1e6:.2f}, wall {(t2 - t0) / K * 1e6:.2f}")
