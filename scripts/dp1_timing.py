"""Step time of a one-rank data-parallel learner (RPL_DP_FORCE=1: NCCL communicator of one rank;
or the peer-memory exchange attached to itself) vs an unattached learner, B = 128."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RPL_DP_FORCE"] = "1"
import torch
import paper_1801_03138_b200.binding as b
from inputs import experiences, init_params
cfg = b.DQNConfig(max_batch=128)
rp = b.Replay(100_000, 27, seed=2)
rp.add_many(experiences(100_000, seed=1))
for mode in ("local", "nccl", "p2p"):
    dqn = b.DQN(cfg, init_params(seed=3))
    if mode == "nccl":
        dqn.attach_nccl(0, 1, b.nccl_unique_id())
    elif mode == "p2p":
        dqn.attach_peers(0, 1, dqn.peer_handle())
    loss = torch.zeros(1, device="cuda")
    for i in range(50):
        dqn.train_step(rp, 128, loss)
    torch.cuda.synchronize()
    l0 = b.kernel_launches()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(2000):
        dqn.train_step(rp, 128, loss)
    e.record()
    torch.cuda.synchronize()
    assert dqn.check() == b.RPL_OK
    print(f"{mode}: {s.elapsed_time(e) / 2000 * 1000:.2f} us/step, {(b.kernel_launches() - l0) / 2000:.2f} launches/step")
    dqn.close()
