"""GPU parity of distinct-index sampling (P:75's planned switch to distinct integers; SURVEY
8(f) NEXT-4; reading Q29: the first B distinct values of the uniform index stream) against
the oracle, through replay_sample and through the train step (fast graph, generic and
byte-state wide paths), with deferred inserts in flight.  Bit-exact indices and batches.
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


@pytest.mark.parametrize("C,B", [(200, 128), (128, 128), (1_000_000, 128), (5000, 4096)])
def test_replay_sample_distinct(b, C, B):
    rp = b.Replay(C, 27, seed=9, sampling="distinct")
    orc = oracle.Ring(C, 27, distinct=True)
    e = experiences(C, seed=4)
    rp.add_many(e)
    orc.add_many(e)
    for _ in range(3):
        g = rp.sample(B)
        rc, o = orc.sample(1, 9, 0, B)
        assert rc == oracle.OK
        g = {k: v.cpu().numpy() for k, v in g.items()}
        assert len(set(g["idx"].tolist())) == B
        for k in ("idx", "s", "s_next", "a", "r", "done"):
            assert np.array_equal(g[k], o[k]), k
    assert rp.check() == b.RPL_OK


def test_distinct_not_ready_below_batch(b):
    rp = b.Replay(100, 27, sampling="distinct")
    rp.add(**experiences(50, seed=1))
    assert rp.sample(64) is None and rp.state()["events"] == 0
    assert rp.sample(50) is not None


def _cfg(b, **kw):
    base = dict(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                double_dqn=True, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=4,
                max_batch=128)
    base.update(kw)
    return b.DQNConfig(**base)


@pytest.mark.parametrize("path", ["fast", "generic"])
def test_train_step_distinct_with_deferred_inserts(b, path, monkeypatch):
    # a 160-slot ring sampled 128 at a time: the uniform stream repeats ~40 rows per batch,
    # the distinct sampler walks past them; 8 host inserts per step are deferred into K1
    if path == "generic":
        monkeypatch.setenv("RPL_PATH", "generic")
    cfg = _cfg(b)
    rp = b.Replay(160, 27, seed=3, burn_in=128, sampling="distinct")
    orc = oracle.Ring(160, 27, distinct=True)
    e = experiences(300, seed=5)
    rp.add(**{k: v[:128] for k, v in e.items()})
    orc.add(**{k: v[:128] for k, v in e.items()})
    dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=6))
    for it in range(12):
        part = {k: v[128 + 8 * it:136 + 8 * it] for k, v in e.items()}
        rp.add(**part)
        orc.add(**part)
        out = step_and_compare(b, cfg, dqn, rp, orc, 128, seed=3, burn_in=128)
        assert out is not None
        assert len(set(dqn.debug(b.RPL_DBG_IDX, 128).tolist())) == 128
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK


def test_wide_u8_step_distinct(b):
    D = 84 * 84 * 4
    cfg = _cfg(b, state_dim=D, double_dqn=False, max_batch=64)
    rp = b.Replay(80, D, seed=21, sampling="distinct", state_dtype="u8")
    orc = oracle.RingU8(80, D, distinct=True)
    e = experiences_u8(80, state_dim=D, seed=22)
    rp.add(**e)
    orc.add(**e)
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=23))
    for _ in range(2):
        step_and_compare(b, cfg, dqn, rp, orc, 64, seed=21)
        assert len(set(dqn.debug(b.RPL_DBG_IDX, 64).tolist())) == 64
