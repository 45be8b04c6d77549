"""Per-phase RPL_TRACE marks of the config-5 wide kernels on a small byte ring (see wide_trace.py)."""
import os, sys
os.environ["RPL_TRACE"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1801_03138_b200.binding as b
from inputs import experiences_u8, init_params
D = 84 * 84 * 4
cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512, double_dqn=False,
                  gamma=0.99, lr=1e-4, huber_kappa=1.0, sync_period=10000, max_batch=256)
rp = b.Replay(2048, D, state_dtype="u8")
e = experiences_u8(1024, seed=1)
rp.add(**e); rp.add(**e)
dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=3))
for _ in range(5):
    dqn.train_step(rp, 256)
torch.cuda.synchronize()
tr = dqn.debug(b.RPL_DBG_TRACE, 256).reshape(-1)[:12]
t = tr.astype(np.int64)
names = ["l0 fwd(skip)", "l0 reduce", "l1 fwd", "-", "head", "bwd l1 pre", "bwd l1", "dz0", "sgd"]
print("phase deltas (us):", [(i, (t[i] - t[i - 1]) / 1000.0) for i in range(1, 10) if t[i] and t[i-1]])
