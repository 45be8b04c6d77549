"""Per-phase timeline of the config-5 tensor-core kernels (RPL_TRACE=1 %globaltimer marks of
wide_l0_kernel / wide_dw0_kernel, averaged over CTAs; times relative to each kernel's first
CTA start).  Run on the GPU box:  python scripts/wide_trace.py"""
import os
import sys

os.environ["RPL_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_03138_b200.binding as b  # noqa: E402
from inputs import experiences_u8, init_params  # noqa: E402

D = 84 * 84 * 4
cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512, double_dqn=False,
                  gamma=0.99, lr=1e-4, huber_kappa=1.0, sync_period=10000, max_batch=256)
rp = b.Replay(4096, D, state_dtype="u8")
e = experiences_u8(1024, seed=1)
for _ in range(4):
    rp.add(**e)
dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=3))
loss = torch.zeros(1, device="cuda")
for _ in range(20):
    dqn.train_step(rp, 256, loss)
torch.cuda.synchronize()
tr = dqn.debug(b.RPL_DBG_TRACE, 256).astype(np.int64)
for k, name, marks in [(4, "wide_l0", {1: "setup", 2: "mainloop+MMA drain", 3: "epilogue"}),
                       (5, "wide_dw0", {1: "setup+db0", 2: "mainloop issue", 4: "MMA drain",
                                        5: "TMEM->smem (+W prefetch)", 6: "SGD epilogue"})]:
    t = tr[k]
    live = t[:, 0] > 0
    t = t[live]
    t0 = t[:, 0].min()
    print(f"{name}: {live.sum()} CTAs, first start -> last end {(t[:, 6 if k == 5 else 3].max() - t0) / 1e3:.2f} us,"
          f" start spread {(t[:, 0].max() - t0) / 1e3:.2f} us")
    prev = 0
    for m, lab in marks.items():
        d = (t[:, m] - t[:, prev]) / 1e3
        print(f"   {lab:28s} mean {d.mean():6.2f} us  max {d.max():6.2f} us")
        prev = m
