"""One-rank peer-memory learner vs an unattached one, step by step: indices of gradient / weight
mismatches (debugging the graph-captured exchange; expects none)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1801_03138_b200.binding as b
from inputs import experiences, init_params
cfg = b.DQNConfig(max_batch=128, sync_period=4, double_dqn=True, lr=1e-3)
p0 = init_params(27, 8, (128,), True, 512, seed=3)
e = experiences(2000, seed=1)
res = []
for attach in (False, True):
    rp = b.Replay(2000, 27, seed=4); rp.add_many(e)
    dqn = b.DQN(cfg, p0)
    if attach:
        dqn.attach_peers(0, 1, dqn.peer_handle())
    loss = torch.zeros(1, device="cuda")
    gs = []
    for s in range(3):
        dqn.train_step(rp, 128, loss); torch.cuda.synchronize()
        gs.append((dqn.get_params(b.RPL_GRAD), dqn.get_params(b.RPL_ONLINE), loss.item()))
    res.append(gs)
for s in range(3):
    g0, g1 = res[0][s][0], res[1][s][0]
    d = np.nonzero(g0 != g1)[0]
    print(f"step {s+1}: grad mismatches {d.size}", (d.min(), d.max()) if d.size else "", "loss", res[0][s][2], res[1][s][2])
    w0, w1 = res[0][s][1], res[1][s][1]
    d = np.nonzero(w0 != w1)[0]
    print(f"   online mismatches {d.size}", (d.min(), d.max()) if d.size else "")
