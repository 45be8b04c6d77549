"""Host-side cost per call of the end-to-end loop (replay_add from host numpy, dqn_train_step
writing the loss into pinned host memory): blocks of 8 steps between synchronisations, so the
calls are timed while the device is behind, not blocked on a full launch queue.
Run on the GPU box:  python scripts/host_costs.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_03138_b200.binding as b  # noqa: E402
from inputs import experiences, init_params  # noqa: E402

cfg = b.DQNConfig(max_batch=128)
rp = b.Replay(100_000, 27, seed=2)
rp.add_many(experiences(100_000, seed=1))
dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=3))
pool = experiences(1024, seed=7)
parts = [{k: v[4 * i:4 * i + 4] for k, v in pool.items()} for i in range(256)]
loss_host = torch.zeros(4096, dtype=torch.float32, pin_memory=True)
views = [loss_host[i:i + 1] for i in range(4096)]
t_add, t_step, t_slice, n = 0.0, 0.0, 0.0, 0
for blk in range(300):
    torch.cuda.synchronize()
    for j in range(8):
        i = blk * 8 + j
        t0 = time.perf_counter()
        rp.add(**parts[i % 256])
        t1 = time.perf_counter()
        lv = loss_host[i % 4096:i % 4096 + 1]
        t2 = time.perf_counter()
        dqn.train_step(rp, 128, lv)
        t3 = time.perf_counter()
        if blk >= 20:
            t_add += t1 - t0
            t_slice += t2 - t1
            t_step += t3 - t2
            n += 1
torch.cuda.synchronize()
print(f"per step over {n} steps: replay_add {1e6 * t_add / n:.2f} us, loss view slice {1e6 * t_slice / n:.2f} us, "
      f"dqn_train_step {1e6 * t_step / n:.2f} us")
# the C calls alone (ctypes, pre-marshalled pointers)
import ctypes as C  # noqa: E402
arrs = [np.ascontiguousarray(parts[0][k]) for k in ("s", "a", "r", "s_next", "done")]
ptrs = [a.ctypes.data_as(C.c_void_p) for a in arrs]
L = b._L
lp = C.c_void_p(views[0].data_ptr())
ta = ts = 0.0
m = 0
for blk in range(300):
    torch.cuda.synchronize()
    for j in range(8):
        t0 = time.perf_counter()
        L.replay_add(rp._h, 4, *ptrs, b.RPL_HOST)
        t1 = time.perf_counter()
        L.dqn_train_step(dqn._h, rp._h, 128, lp)
        t2 = time.perf_counter()
        if blk >= 20:
            ta += t1 - t0
            ts += t2 - t1
            m += 1
torch.cuda.synchronize()
print(f"C calls only: replay_add {1e6 * ta / m:.2f} us, dqn_train_step {1e6 * ts / m:.2f} us")
