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


# ---- RPL_RING_HOST_BATCH: the paper's in-RAM replay ("copies sampled batches to the
# GPU"): CPU ring, CPU sampler, CPU gather, one H2D batch copy per step ----------------

def test_host_batch_sample_matches_oracle(b):
    C, B = 1000, 128
    rp = b.Replay(C, 27, seed=9, ring_memory="host_batch", burn_in=50)
    orc = oracle.Ring(C, 27)
    e = experiences(C + 77, seed=4)
    assert rp.sample(B) is None   # burn-in: nothing sampled, no event consumed
    for part in (slice(0, 250), slice(250, C + 77)):
        rp.add(**{k: v[part] for k, v in e.items()})
        orc.add(**{k: v[part] for k, v in e.items()})
    st = rp.state()
    assert (st["cursor"], st["size"], st["total"], st["h2d_bytes"]) == (orc.cursor, orc.size, orc.total, 0)
    for ev in range(3):
        g = rp.sample(B)
        rc, o = orc.sample(50, 9, 0, B)
        assert rc == oracle.OK
        g = {k: v.cpu().numpy() for k, v in g.items()}
        for k in ("idx", "s", "s_next", "a", "r", "done"):
            assert np.array_equal(g[k], o[k]), k
    # each sample crossed PCIe as the batch tensors: B * (2 * 27 * 4 + 9) bytes
    assert rp.state()["h2d_bytes"] == 3 * B * (2 * 27 * 4 + 9)
    with pytest.raises(b.RplError):
        import torch
        rp.gather(torch.arange(4, dtype=torch.int32, device="cuda"))
    with pytest.raises(b.RplError):   # device-sourced adds: the in-RAM replay takes host inputs
        import torch
        rp.add(**{k: torch.from_numpy(v[:3]).cuda() for k, v in e.items()})
    assert rp.check() == b.RPL_OK


@pytest.mark.parametrize("ddqn", [False, True], ids=["dqn", "ddqn"])
def test_host_batch_train_step(b, ddqn):
    # the fast kernels on the CPU-gathered batch: bit-exact batch, 1e-5 results, B ragged and
    # beyond a 16-row tile; adds interleaved (the CPU writes the host rows); the step's one
    # transfer is B * (256 + 4) bytes
    cfg = b.DQNConfig(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=ddqn, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=3,
                      max_batch=300)
    rp = b.Replay(400, 27, seed=3, burn_in=128, ring_memory="host_batch")
    orc = oracle.Ring(400, 27)
    e = experiences(700, seed=5)
    rp.add(**{k: v[:200] for k, v in e.items()})
    orc.add(**{k: v[:200] for k, v in e.items()})
    dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=6))
    h0 = rp.state()["h2d_bytes"]
    batches = [128, 37, 300, 1, 128, 77]
    for it, B in enumerate(batches):
        part = {k: v[200 + 40 * it:240 + 40 * it] for k, v in e.items()}
        rp.add(**part)
        orc.add(**part)
        assert step_and_compare(b, cfg, dqn, rp, orc, B, seed=3, burn_in=128) is not None
    assert rp.state()["h2d_bytes"] - h0 == sum(batches) * (256 + 4)
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK


def test_host_batch_equals_device_ring_training(b):
    # the two replays hold the same experiences and draw the same Philox stream: 20 train
    # steps from the in-RAM replay and from the HBM ring give bit-identical parameters
    cfg = b.DQNConfig(max_batch=128, sync_period=5, double_dqn=True, lr=1e-3)
    p0 = init_params(27, 8, (128,), True, 512, seed=8)
    e = experiences(3000, seed=9)
    out = []
    for mem in ("device", "host_batch"):
        rp = b.Replay(2000, 27, seed=4, ring_memory=mem)
        rp.add_many({k: v[:2000] for k, v in e.items()})
        dqn = b.DQN(cfg, p0)
        for it in range(20):
            rp.add(**{k: v[2000 + 8 * it:2008 + 8 * it] for k, v in e.items()})
            assert dqn.train_step(rp, 128) == b.RPL_OK
        out.append((dqn.get_params(b.RPL_ONLINE), dqn.get_params(b.RPL_TARGET)))
        assert dqn.check() == b.RPL_OK
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("ddqn", [False, True], ids=["dqn", "ddqn"])
def test_host_batch_tcgen05_step(b, ddqn):
    # the CPU-gathered batch into the large-batch tcgen05 step (tc_big.cuh T0 reads the copied
    # rows): bit-exact batch, 1e-5 results at B = 700 (ragged) and 1024
    cfg = b.DQNConfig(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=ddqn, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=2,
                      max_batch=1024)
    rp = b.Replay(3000, 27, seed=7, ring_memory="host_batch")
    orc = oracle.Ring(3000, 27)
    e = experiences(3000, seed=15)
    rp.add(**e)
    orc.add(**e)
    dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=16))
    for B in (700, 1024, 700):
        assert step_and_compare(b, cfg, dqn, rp, orc, B, seed=7) is not None
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK


@pytest.mark.parametrize("B", [128, 700])
def test_host_batch_distinct_sampling(b, B):
    # the paper's in-RAM replay drew its batches with random.sample (without replacement):
    # RPL_RING_HOST_BATCH with distinct sampling -- the CPU takes the first B distinct values of
    # the uniform Philox stream (reading Q29), bit-exact against the oracle's distinct ring, and
    # the train step (mma.sync at 128, tcgen05 at 700) within 1e-5
    cfg = b.DQNConfig(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=True, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=2,
                      max_batch=1024)
    rp = b.Replay(1500, 27, seed=9, ring_memory="host_batch", sampling="distinct")
    orc = oracle.Ring(1500, 27, distinct=True)
    e = experiences(1500, seed=17)
    rp.add(**e)
    orc.add(**e)
    dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=18))
    for _ in range(3):
        assert step_and_compare(b, cfg, dqn, rp, orc, B, seed=9) is not None
    idx = dqn.debug(b.RPL_DBG_IDX, B)
    assert len(set(idx.tolist())) == B
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK
