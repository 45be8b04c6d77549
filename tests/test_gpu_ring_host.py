"""GPU parity of the in-RAM comparison mode: the ring's
rows in pinned, device-mapped host memory, read by the same kernels across PCIe.  Sampling,
gathering and the train step must give exactly what the oracle (and the HBM ring) gives:
bit-exact indices and batches, FP32 results within the parity tolerance.
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


@pytest.mark.parametrize("C,B,distinct", [(1000, 128, False), (300, 64, True)])
def test_host_ring_sample_matches_oracle(b, C, B, distinct):
    rp = b.Replay(C, 27, seed=9, ring_memory="host", sampling="distinct" if distinct else "uniform")
    orc = oracle.Ring(C, 27, distinct=distinct)
    e = experiences(C + 77, seed=4)     # wraps the ring
    for part in (slice(0, 250), slice(250, C + 77)):
        rp.add(**{k: v[part] for k, v in e.items()})
        orc.add(**{k: v[part] for k, v in e.items()})
    for _ in range(3):
        g = rp.sample(B)
        rc, o = orc.sample(1, 9, 0, B)
        assert rc == oracle.OK
        g = {k: v.cpu().numpy() for k, v in g.items()}
        for k in ("idx", "s", "s_next", "a", "r", "done"):
            assert np.array_equal(g[k], o[k]), k
    assert rp.check() == b.RPL_OK


@pytest.mark.parametrize("path", ["fast", "generic"])
def test_host_ring_train_step(b, path, monkeypatch):
    # the fast graph (gather fused into K1, deferred inserts written by K3 into host rows) and
    # the cooperative kernel, each reading its batch across PCIe
    if path == "generic":
        monkeypatch.setenv("RPL_PATH", "generic")
    cfg = b.DQNConfig(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=True, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=3,
                      max_batch=128)
    rp = b.Replay(400, 27, seed=3, burn_in=128, ring_memory="host")
    orc = oracle.Ring(400, 27)
    e = experiences(600, seed=5)
    rp.add(**{k: v[:200] for k, v in e.items()})
    orc.add(**{k: v[:200] for k, v in e.items()})
    dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=6))
    for it in range(8):
        part = {k: v[200 + 16 * it:216 + 16 * it] for k, v in e.items()}
        rp.add(**part)
        orc.add(**part)
        assert step_and_compare(b, cfg, dqn, rp, orc, 128 if it % 2 else 37, seed=3, burn_in=128) is not None
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK


def test_host_ring_byte_states(b):
    # config-5-shaped byte states from a host ring through the tensor-core layer 0
    D = 84 * 84 * 4
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=False, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=2,
                      max_batch=64)
    rp = b.Replay(96, D, seed=11, state_dtype="u8", ring_memory="host")
    orc = oracle.RingU8(96, D)
    e = experiences_u8(96, state_dim=D, seed=12)
    rp.add(**e)
    orc.add(**e)
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=13))
    for batch in (64, 9):
        step_and_compare(b, cfg, dqn, rp, orc, batch, seed=11)
    assert dqn.check() == b.RPL_OK
