"""Config-5 step time (84x84x4 bytes, B = 256, 4,096-row byte ring) of an unattached learner and
of a one-rank peer-memory data-parallel learner (the exchange's reduce-scatter kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03138_b200.binding as b
from inputs import experiences_u8, init_params
D = 84 * 84 * 4
cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512, max_batch=256,
                  sync_period=100, lr=1e-4)
rp = b.Replay(4096, D, seed=2, state_dtype="u8")
e = experiences_u8(1024, state_dim=D, seed=1)
for i in range(4):
    rp.add(**e)
for mode in ("local", "p2p"):
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=3))
    if mode == "p2p":
        dqn.attach_peers(0, 1, dqn.peer_handle())
    loss = torch.zeros(1, device="cuda")
    for i in range(20):
        dqn.train_step(rp, 256, loss)
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(300):
        dqn.train_step(rp, 256, loss)
    t.record()
    torch.cuda.synchronize()
    assert dqn.check() == b.RPL_OK
    print(f"c5 {mode}: {s.elapsed_time(t) / 300 * 1000:.2f} us/step")
    dqn.close()
