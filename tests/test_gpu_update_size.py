"""GPU parity of P:73's block updates (the update-size queue): host
experiences wait in a queue until update_size of them form a block, which is one insert (one
H2D transfer); queued experiences are not part of the replay.  Checked against the oracle's
queue (oracle_queue_*, pinned in tests/test_oracle_replay.py): bit-exact ring state, rows,
samples and byte accounting, and a train step over a queued replay.
"""
import numpy as np
import pytest

import oracle
from inputs import experiences, init_params
from parity import step_and_compare

pytestmark = pytest.mark.gpu

ROW_BYTES = 2 * 27 * 4 + 4 + 4 + 1   # one host experience crossing PCIe (s, s', a, r, done)


@pytest.fixture(scope="module")
def b():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1801_03138_b200.binding as binding
    return binding


def _same_state(rp, orc):
    st = rp.state()
    assert (st["cursor"], st["size"], st["total"]) == (orc.cursor, orc.size, orc.total)
    assert rp.queued == orc.queued


def test_queue_blocks_match_oracle(b):
    import torch
    C, U = 12, 4
    rp = b.Replay(C, 27, seed=5, update_size=U)
    orc = oracle.Ring(C, 27, update_size=U)
    e = experiences(200, seed=31)
    t = 0
    for step, k in enumerate([1, 2, 3, 4, 9, 1, 12, 5, 3, 0, 7, 2, 11]):
        part = {kk: v[t:t + k] for kk, v in e.items()}
        t += k
        rp.add(**part)
        assert orc.add(**part) == oracle.OK
        if step % 4 == 3:
            assert rp.flush_queue() == orc.flush_queue()
        _same_state(rp, orc)
        if orc.size:
            idx = torch.arange(orc.size, dtype=torch.int32, device="cuda")
            g = {kk: v.cpu().numpy() for kk, v in rp.gather(idx).items()}
            o = orc.gather(np.arange(orc.size, dtype=np.int32))
            for kk in ("s", "s_next", "a", "r", "done"):
                assert np.array_equal(g[kk], o[kk]), kk
    for _ in range(3):
        g = rp.sample(64)
        rc, o = orc.sample(1, 5, 0, 64)
        assert rc == oracle.OK
        for kk in ("idx", "s", "s_next", "a", "r", "done"):
            assert np.array_equal(g[kk].cpu().numpy(), o[kk]), kk
    assert rp.check() == b.RPL_OK


def test_update_size_2000_is_one_transfer(b):
    # P:119's update-size 2,000: 1,999 single adds cross nothing; the 2,000th writes the block
    # in one H2D transfer of 2,000 experiences
    rp = b.Replay(10_000, 27, update_size=2000)
    e = experiences(2000, seed=32)
    for i in range(1999):
        rp.add(**{k: v[i:i + 1] for k, v in e.items()})
    st = rp.state()
    assert st["size"] == 0 and st["h2d_bytes"] == 0 and rp.queued == 1999
    assert rp.sample(8) is None   # nothing sampleable yet
    rp.add(**{k: v[1999:] for k, v in e.items()})
    st = rp.state()
    assert st["size"] == 2000 and rp.queued == 0 and st["h2d_bytes"] == 2000 * ROW_BYTES
    orc = oracle.Ring(10_000, 27)
    orc.add(**e)
    g = rp.sample(256)
    rc, o = orc.sample(1, 2, 0, 256)
    for k in ("idx", "s", "s_next", "a", "r", "done"):
        assert np.array_equal(g[k].cpu().numpy(), o[k]), k


def test_queue_rejects_device_adds_and_bad_done(b):
    import torch
    rp = b.Replay(100, 27, update_size=10)
    e = experiences(5, seed=33)
    with pytest.raises(b.RplError):
        rp.add(**{k: torch.from_numpy(v).cuda() for k, v in e.items()})
    bad = dict(e, done=np.array([0, 0, 2, 0, 0], np.uint8))
    with pytest.raises(b.RplError):
        rp.add(**bad)
    assert rp.queued == 0


def test_train_step_over_a_queued_replay(b):
    # the learner only ever sees written blocks; queued experiences stay out of every batch
    cfg = b.DQNConfig(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=False, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=5,
                      max_batch=64)
    rp = b.Replay(500, 27, seed=3, burn_in=64, update_size=50)
    orc = oracle.Ring(500, 27, update_size=50)
    e = experiences(700, seed=34)
    dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=6))
    t = 0
    for it in range(10):
        k = 23 + 7 * (it % 3)
        part = {kk: v[t:t + k] for kk, v in e.items()}
        t += k
        rp.add(**part)
        orc.add(**part)
        _same_state(rp, orc)
        out = step_and_compare(b, cfg, dqn, rp, orc, 64, seed=3, burn_in=64)
        assert (out is None) == (orc.size < 64)
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK
