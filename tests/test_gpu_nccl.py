"""The NCCL data-parallel path of dqn_train_step on one GPU (RPL_DP_FORCE=1 builds a
communicator of one rank): the library loads NCCL, creates the communicator from a unique id,
all-reduces (mean) the gradient + loss word every step and applies the SGD after it
(P:144), or averages the parameters every K steps (reading Q31).  Over a single rank the
means are identities, so the parameters must equal an unattached learner's bit for bit.
"""
import numpy as np
import pytest

from inputs import experiences, init_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1801_03138_b200.binding as binding
    return binding


@pytest.mark.parametrize("avg_period", [0, 3])
@pytest.mark.parametrize("net", ["fast", "generic"])
def test_nccl_single_rank_equals_local(b, monkeypatch, avg_period, net):
    import torch
    if net == "generic":
        monkeypatch.setenv("RPL_PATH", "generic")
    cfg = b.DQNConfig(max_batch=128, sync_period=4, avg_period=avg_period, double_dqn=True,
                      lr=1e-3)
    p0 = init_params(27, 8, (128,), True, 512, seed=3)
    e = experiences(2000, seed=1)
    runs = []
    for attach in (False, True):
        monkeypatch.setenv("RPL_DP_FORCE", "1" if attach else "0")
        rp = b.Replay(2000, 27, seed=4)
        rp.add_many(e)
        dqn = b.DQN(cfg, p0)
        if attach:
            dqn.attach_nccl(0, 1, b.nccl_unique_id())
        loss = torch.zeros(1, device="cuda")
        for _ in range(7):
            assert dqn.train_step(rp, 128, loss) == b.RPL_OK
        torch.cuda.synchronize()
        assert dqn.check() == b.RPL_OK and np.isfinite(loss.item())
        runs.append((dqn.get_params(b.RPL_ONLINE), dqn.get_params(b.RPL_TARGET), loss.item()))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])
    assert runs[0][2] == runs[1][2]


def test_nccl_graph_captured_exchange_loss_destinations(b, monkeypatch):
    # the NCCL all-reduce and the SGD after it are captured in the step graph (one launch per
    # step); the SGD kernel writes the mean loss to the caller's destination, which may change
    # between steps (device, pinned host): a one-rank learner must equal an unattached one
    import torch
    cfg = b.DQNConfig(max_batch=128, sync_period=3, double_dqn=True, lr=1e-3)
    p0 = init_params(27, 8, (128,), True, 512, seed=5)
    e = experiences(2000, seed=6)
    runs = []
    for attach in (False, True):
        monkeypatch.setenv("RPL_DP_FORCE", "1" if attach else "0")
        rp = b.Replay(2000, 27, seed=7)
        rp.add_many(e)
        dqn = b.DQN(cfg, p0)
        if attach:
            dqn.attach_nccl(0, 1, b.nccl_unique_id())
        dev = torch.zeros(1, device="cuda")
        host = torch.zeros(6, dtype=torch.float32, pin_memory=True)
        losses = []
        for i in range(6):
            dst = host[i:i + 1] if i % 2 else dev
            assert dqn.train_step(rp, 128, dst) == b.RPL_OK
            torch.cuda.synchronize()
            losses.append(float(dst.cpu()[0]) if dst is dev else float(dst[0]))
        assert dqn.check() == b.RPL_OK
        runs.append((dqn.get_params(b.RPL_ONLINE), dqn.get_params(b.RPL_TARGET), losses))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])
    assert runs[0][2] == runs[1][2]


def test_nccl_single_rank_wide_learner_equals_local(b, monkeypatch):
    # config-5 network (tcgen05 layer 0): the SGD after the all-reduce rewrites W0 and its bf16
    # planes (the target's on sync steps), which the next step's layer 0 reads
    from inputs import experiences_u8
    D = 84 * 84 * 4
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      max_batch=32, sync_period=3, lr=1e-3)
    p0 = init_params(D, 8, (128,), True, 512, seed=13)
    e = experiences_u8(64, state_dim=D, seed=12)
    runs = []
    for attach in (False, True):
        monkeypatch.setenv("RPL_DP_FORCE", "1" if attach else "0")
        rp = b.Replay(64, D, seed=11, state_dtype="u8")
        rp.add(**e)
        dqn = b.DQN(cfg, p0)
        if attach:
            dqn.attach_nccl(0, 1, b.nccl_unique_id())
        for _ in range(7):
            assert dqn.train_step(rp, 32) == b.RPL_OK
        assert dqn.check() == b.RPL_OK
        runs.append((dqn.get_params(b.RPL_ONLINE), dqn.get_params(b.RPL_TARGET)))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])
