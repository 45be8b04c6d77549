import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1801_03138_b200.binding as b
from inputs import experiences, init_params
cfg = b.DQNConfig(max_batch=128)
rp = b.Replay(1_000_000, 27, seed=2)
rp.add_many(experiences(1_000_000, seed=1))
dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=3))
pool = experiences(1024, seed=7)
parts_h = [{k: v[4 * i:4 * i + 4] for k, v in pool.items()} for i in range(256)]
pool_d = {k: torch.from_numpy(v).cuda() for k, v in pool.items()}
parts_d = [{k: v[4 * i:4 * i + 4] for k, v in pool_d.items()} for i in range(256)]
K = 5000
loss_dev = torch.zeros(1, device="cuda")
loss_host = torch.zeros(K, dtype=torch.float32, pin_memory=True)
slots = [loss_host[i:i + 1] for i in range(K)]
st = torch.cuda.current_stream()
for name, host_add, host_loss in [("dev add, dev loss", False, False), ("host add, dev loss", True, False),
                                  ("dev add, host loss", False, True), ("host add, host loss", True, True)]:
    for rep in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.record(st)
        for i in range(K):
            if host_add:
                rp.add(**parts_h[i % 256])
            else:
                rp.add(**parts_d[i % 256], defer=True)
            dqn.train_step(rp, 128, slots[i] if host_loss else loss_dev)
        e.record(st)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    print(f"{name:22s} device {1000 * s.elapsed_time(e) / K:6.2f} us/step  wall {1e6 * wall / K:6.2f}")
os._exit(0)
