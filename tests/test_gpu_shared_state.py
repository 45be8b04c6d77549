"""GPU parity of shared-state storage ("by only storing one state per experience,
and modifying the sample operations, the in-GPU experience replay could decrease the required
GPU memory size by a factor of two"; reading Q30) against the oracle:
half-width rows, the new state read from the next slot, the sampler over all but the newest
experience -- through replay_sample, the fast graph (with deferred inserts), the generic and
the byte-state wide paths.  Indices and batches bit-exact, the step within 1e-5.
"""
import numpy as np
import pytest

import oracle
from inputs import experiences, experiences_u8, init_params
from parity import step_and_compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1801_03138_b200.binding as binding
    return binding


def _add(rp, orc, part, device=False):
    import torch
    if device:
        rp.add(**{k: torch.from_numpy(v).cuda() for k, v in part.items() if k != "s_next"},
               s_next=None)
    else:
        rp.add(part["s"], part["a"], part["r"], None, part["done"])
    assert orc.add(part["s"], part["a"], part["r"], None, part["done"]) == oracle.OK


@pytest.mark.parametrize("distinct", [False, True])
def test_shared_state_sample_wraps(b, distinct):
    C, D, B = 64, 27, 32
    rp = b.Replay(C, D, seed=5, sampling="distinct" if distinct else "uniform", shared_state=True)
    orc = oracle.Ring(C, D, distinct=distinct, shared=True)
    e = experiences(400, seed=8)
    t = 0
    for i, k in enumerate([1, 20, 13, 40, 64, 9, 31, 50]):
        _add(rp, orc, {kk: v[t:t + k] for kk, v in e.items()}, device=bool(i % 2))
        t += k
        g = rp.sample(B)
        rc, o = orc.sample(1, 5, 0, B)
        if rc == oracle.NOT_READY:
            assert g is None
            continue
        g = {kk: v.cpu().numpy() for kk, v in g.items()}
        for kk in ("idx", "s", "s_next", "a", "r", "done"):
            assert np.array_equal(g[kk], o[kk]), kk
    # one state per experience crossed PCIe
    assert rp.state()["h2d_bytes"] == sum([1, 13, 64, 31]) * (4 * D + 9)
    assert rp.check() == b.RPL_OK


@pytest.mark.parametrize("distinct", [False, True])
@pytest.mark.parametrize("path", ["fast", "generic"])
def test_shared_state_train_step(b, path, distinct, monkeypatch):
    # a 160-slot ring that wraps during the run, 8 host inserts per step deferred into the step
    # (the s' of the newest committed slot is read through from the pending insert); with the
    # distinct sampler the 128 distinct experiences come from the 159 sampleable ones
    if path == "generic":
        monkeypatch.setenv("RPL_PATH", "generic")
    cfg = b.DQNConfig(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=True, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=3,
                      max_batch=128)
    rp = b.Replay(160, 27, seed=3, shared_state=True,
                  sampling="distinct" if distinct else "uniform")
    orc = oracle.Ring(160, 27, shared=True, distinct=distinct)
    e = experiences(400, seed=6)
    _add(rp, orc, {k: v[:140] for k, v in e.items()})
    dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=7))
    for it in range(10):
        _add(rp, orc, {k: v[140 + 8 * it:148 + 8 * it] for k, v in e.items()})
        assert step_and_compare(b, cfg, dqn, rp, orc, 128, seed=3) is not None
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK


def test_shared_state_wide_u8(b):
    D = 84 * 84 * 4
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=False, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=0,
                      max_batch=64)
    rp = b.Replay(70, D, seed=21, state_dtype="u8", shared_state=True)
    orc = oracle.RingU8(70, D, shared=True)
    e = experiences_u8(90, state_dim=D, seed=22)
    _add(rp, orc, {k: v[:90] for k, v in e.items()} if False else {k: v[:70] for k, v in e.items()})
    _add(rp, orc, {k: v[70:90] for k, v in e.items()})   # wraps: oldest slot = cursor
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=23))
    for _ in range(2):
        step_and_compare(b, cfg, dqn, rp, orc, 64, seed=21)
