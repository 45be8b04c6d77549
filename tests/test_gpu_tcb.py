"""GPU parity of the large-batch tensor-core step (csrc/tc_big.cuh: batches >= kTcbMinBatch = 640)
against the oracle, through the C-ABI (tests/parity.py: idx / batch bit-exact, Q / y / loss /
gradients / new weights within 1e-5 normwise in FP32, 2e-2 at BF16 precision).

Covers: DQN and Double DQN, full and ragged 128-row tiles, several teacher-forced steps with
target syncs (the W1 images K4 writes for the next step), a plain MLP head, deferred inserts
read through, distinct sampling, shared-state storage, switching between batch sizes that take
the mma.sync and the tensor-core kernels (the W1 image refresh), BF16 precision.
"""
import numpy as np
import pytest

import oracle
from inputs import experiences, init_params
from parity import step_and_compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1801_03138_b200.binding as binding
    return binding


def _cfg(b, **kw):
    base = dict(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                double_dqn=False, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=2,
                max_batch=4096)
    base.update(kw)
    return b.DQNConfig(**base)


def _params(cfg, seed=3):
    return init_params(cfg.state_dim, cfg.n_actions, cfg.hidden, cfg.dueling, cfg.stream, seed=seed)


def _replay(b, cap=20_000, n=25_000, seed=6, **kw):
    rp = b.Replay(cap, 27, seed=5, rank=1, **kw)
    orc = oracle.Ring(cap, 27, distinct=kw.get("sampling") == "distinct", shared=kw.get("shared_state", False))
    e = experiences(n, seed=seed, done_prob=0.1)
    rp.add_many(e)
    orc.add_many(e)
    return rp, orc


@pytest.mark.parametrize("ddqn", [False, True], ids=["dqn", "ddqn"])
@pytest.mark.parametrize("batch", [640, 700, 1000, 4096])
def test_tcb_steps(b, batch, ddqn):
    cfg = _cfg(b, double_dqn=ddqn)
    rp, orc = _replay(b)
    dqn = b.DQN(cfg, _params(cfg, seed=7))
    for _ in range(3):   # sync_period 2: the target image is rewritten by K4 on step 2
        assert step_and_compare(b, cfg, dqn, rp, orc, batch, seed=5, rank=1) is not None
    assert dqn.check() == b.RPL_OK


def test_tcb_plain_mlp(b):
    cfg = _cfg(b, dueling=False, hidden=(128, 256), double_dqn=True, max_batch=1024)
    rp, orc = _replay(b)
    dqn = b.DQN(cfg, init_params(27, 8, (128, 256), False, 0, seed=9))
    for _ in range(2):
        assert step_and_compare(b, cfg, dqn, rp, orc, 777, seed=5, rank=1) is not None


def test_tcb_switching_batch_sizes(b):
    # mma.sync steps (B < 640) update W1 without its image; the next tensor-core step re-splits
    cfg = _cfg(b, double_dqn=True, sync_period=3)
    rp, orc = _replay(b)
    dqn = b.DQN(cfg, _params(cfg, seed=11))
    for batch in (128, 1024, 64, 700, 4096, 300, 512):
        assert step_and_compare(b, cfg, dqn, rp, orc, batch, seed=5, rank=1) is not None
    dqn.sync_target()
    orc_t = dqn.get_params(b.RPL_ONLINE)
    assert np.array_equal(dqn.get_params(b.RPL_TARGET), orc_t)
    assert step_and_compare(b, cfg, dqn, rp, orc, 1024, seed=5, rank=1) is not None


@pytest.mark.parametrize("mode", ["host", "device_defer"])
def test_tcb_deferred_insert(b, mode):
    import torch
    cfg = _cfg(b, double_dqn=True)
    rp, orc = _replay(b, cap=3000, n=2500)
    dqn = b.DQN(cfg, _params(cfg, seed=13))
    for step in range(4):
        e = experiences(700, seed=100 + step, done_prob=0.1)
        if mode == "host":
            rp.add(**e)
        else:
            rp.add(**{k: torch.from_numpy(v).cuda() for k, v in e.items()}, defer=True)
        orc.add(**e)
        assert step_and_compare(b, cfg, dqn, rp, orc, 1024, seed=5, rank=1) is not None
    # the ring rows the steps wrote for the deferred inserts
    st = rp.state()
    assert st["size"] == 3000


def test_tcb_distinct_and_shared(b):
    cfg = _cfg(b, double_dqn=True)
    rp, orc = _replay(b, sampling="distinct")
    dqn = b.DQN(cfg, _params(cfg, seed=17))
    assert step_and_compare(b, cfg, dqn, rp, orc, 1000, seed=5, rank=1) is not None
    rp2, orc2 = _replay(b, shared_state=True)
    dqn2 = b.DQN(cfg, _params(cfg, seed=19))
    assert step_and_compare(b, cfg, dqn2, rp2, orc2, 1000, seed=5, rank=1) is not None


@pytest.mark.parametrize("ddqn", [False, True], ids=["dqn", "ddqn"])
def test_tcb_bf16_precision(b, ddqn):
    cfg = _cfg(b, double_dqn=ddqn, precision="bf16")
    rp, orc = _replay(b)
    dqn = b.DQN(cfg, _params(cfg, seed=21))
    for _ in range(2):
        assert step_and_compare(b, cfg, dqn, rp, orc, 2048, seed=5, rank=1, tol=2e-2) is not None
