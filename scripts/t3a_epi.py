"""T3a epilogue phases (experiment build -DRPL_T3A_EPI_TRACE, RPL_TRACE=1): cycles since CTA start."""
import os, sys
import numpy as np
os.environ["RPL_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03138_b200.binding as b
from inputs import experiences, init_params
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = b.DQNConfig(max_batch=B, double_dqn=True)
rp = b.Replay(1_000_000, 27, seed=2); rp.add_many(experiences(1_000_000, seed=1))
dqn = b.DQN(cfg, init_params(seed=3)); loss = torch.zeros(1, device="cuda")
for _ in range(20): dqn.train_step(rp, B, loss)
torch.cuda.synchronize()
tr = dqn.debug(b.RPL_DBG_TRACE, B).astype(np.int64)[5]
m = tr[:, 0] > 0
dur = (tr[m, 1] - tr[m, 0]) / 1000.0
lo, sh, pw = tr[m, 5] / 1965.0, tr[m, 6] / 1965.0, tr[m, 7] / 1965.0
print(f"B={B}: CTA {dur.mean():.2f} us; loop done {lo.mean():.2f}; shuffles {(sh - lo).mean():.2f}; partial writes {(pw - sh).mean():.2f}; dW1 out {(dur - pw).mean():.2f} (max {(dur - pw).max():.2f})")
