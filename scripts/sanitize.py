"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
kernel family of the library once or twice on small shapes -- replay insert / sample / gather
(fp32, u8, shared states, distinct), the fast train-step graph (DQN, DDQN, deferred host and
device inserts), the cooperative generic step, the config-5 wide step on tcgen05 (graph and
non-graph), reduced precision.  Usage on the GPU box:
    compute-sanitizer --tool memcheck python scripts/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_03138_b200.binding as b  # noqa: E402
from inputs import experiences, experiences_u8, init_params  # noqa: E402


def run_fast(ddqn, precision="fp32", sampling="uniform", shared=False):
    cfg = b.DQNConfig(max_batch=128, double_dqn=ddqn, sync_period=2, precision=precision)
    rp = b.Replay(600, 27, seed=3, sampling=sampling, shared_state=shared)
    e = experiences(700, seed=4)
    rp.add(**{k: v[:500] for k, v in e.items()})
    dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=5))
    loss = torch.zeros(1, device="cuda")
    for i in range(3):
        rp.add(**{k: v[500 + 8 * i:508 + 8 * i] for k, v in e.items()})   # deferred host insert
        assert dqn.train_step(rp, 128 if i != 1 else 37, loss) == b.RPL_OK
    ed = {k: torch.from_numpy(v[600:604]).cuda() for k, v in e.items()}
    rp.add(**ed, defer=True)
    assert dqn.train_step(rp, 64, loss) == b.RPL_OK
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK
    g = rp.sample(64)
    rp.gather(g["idx"])
    torch.cuda.synchronize()


def run_wide(graph=True):
    D = 84 * 84 * 4
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      max_batch=32, sync_period=2)
    rp = b.Replay(64, D, seed=11, state_dtype="u8")
    rp.add(**experiences_u8(64, state_dim=D, seed=12))
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=13))
    for bs in (32, 7):
        assert dqn.train_step(rp, bs) == b.RPL_OK
    assert dqn.check() == b.RPL_OK


what = sys.argv[1:] or ["fast", "ddqn", "bf16", "distinct", "shared", "generic", "wide", "wide-nograph"]
for w in what:
    if w == "fast":
        run_fast(False)
    elif w == "ddqn":
        run_fast(True)
    elif w == "bf16":
        run_fast(False, precision="bf16")
    elif w == "distinct":
        run_fast(False, sampling="distinct")
    elif w == "shared":
        run_fast(True, shared=True)
    elif w == "generic":
        os.environ["RPL_PATH"] = "generic"
        run_fast(True)
        del os.environ["RPL_PATH"]
    elif w == "wide":
        run_wide()
    elif w == "wide-nograph":
        os.environ["RPL_NO_GRAPH"] = "1"
        run_wide()
        del os.environ["RPL_NO_GRAPH"]
    print("ok", w, flush=True)
print("sanitize workload done")
os._exit(0)
