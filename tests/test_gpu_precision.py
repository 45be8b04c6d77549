"""Reduced-precision learners (rpl_dqn_config.precision; SURVEY 8(a) A5 "BF16 MMA (fast)", 8(d)
D1 / D4 "FP32 and BF16"): one tensor-core product of tf32- or bf16-rounded operands instead of
the FP32-accurate splits.  Parity against the fp64 oracle at the north star's BF16 tolerance
(2e-2 normwise, teacher-forced per step; ReLU / argmax decisions replayed within it), and a
check that the mode really changes the arithmetic.
"""
import numpy as np
import pytest

import oracle
from inputs import experiences, experiences_u8, init_params
from parity import step_and_compare

pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module")
def b():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1801_03138_b200.binding as binding
    return binding


@pytest.mark.parametrize("precision", ["tf32", "bf16"])
@pytest.mark.parametrize("ddqn", [False, True])
def test_reduced_precision_fast_path(b, precision, ddqn):
    cfg = b.DQNConfig(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=ddqn, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=3,
                      max_batch=256, precision=precision)
    rp = b.Replay(2000, 27, seed=4)
    orc = oracle.Ring(2000, 27)
    e = experiences(2000, seed=41)
    rp.add(**e)
    orc.add(**e)
    dqn = b.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=42))
    for batch in (128, 37, 256, 128):
        assert step_and_compare(b, cfg, dqn, rp, orc, batch, seed=4, tol=TOL) is not None
    assert dqn.check() == b.RPL_OK


def test_reduced_precision_changes_the_products(b):
    # the same weights and batch: FP32 mode matches the oracle to 1e-5, BF16 mode does not
    # match FP32 bit for bit (the correction products are really dropped)
    e = experiences(1000, seed=43)
    params = init_params(27, 8, (128,), True, 512, seed=44)
    q = {}
    for prec in ("fp32", "bf16"):
        cfg = b.DQNConfig(max_batch=128, precision=prec)
        rp = b.Replay(1000, 27, seed=5)
        rp.add(**e)
        dqn = b.DQN(cfg, params)
        dqn.train_step(rp, 128)
        q[prec] = dqn.debug(b.RPL_DBG_Q, 128)
    assert not np.array_equal(q["fp32"], q["bf16"])
    err = np.max(np.abs(q["fp32"] - q["bf16"])) / np.max(np.abs(q["fp32"]))
    assert 1e-6 < err < TOL


@pytest.mark.parametrize("precision", ["tf32", "bf16"])
def test_reduced_precision_wide_layer0(b, precision):
    # config-5 network: layer 0 with 2 (tf32) or 1 (bf16) bf16 terms of the fp32 operands
    D = 84 * 84 * 4
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=False, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=2,
                      max_batch=64, precision=precision)
    rp = b.Replay(96, D, seed=11, state_dtype="u8")
    orc = oracle.RingU8(96, D)
    e = experiences_u8(96, state_dim=D, seed=12)
    rp.add(**e)
    orc.add(**e)
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=13))
    for batch in (64, 9, 64):
        step_and_compare(b, cfg, dqn, rp, orc, batch, seed=11, tol=TOL)
    assert dqn.check() == b.RPL_OK


def test_precision_is_validated(b):
    with pytest.raises(KeyError):
        b.DQNConfig(precision="fp8")._c()
