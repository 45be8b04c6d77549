"""GPU parity of the fused train step (dqn_train_step through the C-ABI) against the oracle.

Teacher-forced per step (tests/parity.py): idx and gathered batch bit-exact; Q, y, loss,
gradients and new weights within 1e-5 normwise in FP32 (BASELINE north star); bit-exact in
the dyadic exact-input mode.
"""
import math

import numpy as np
import pytest

import oracle
from inputs import experiences, init_params
from parity import f32, normwise, oracle_net, step_and_compare

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
                double_dqn=False, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=0,
                max_batch=4096)
    base.update(kw)
    return b.DQNConfig(**base)


def _params(cfg, seed=3, dyadic=False):
    return init_params(cfg.state_dim, cfg.n_actions, cfg.hidden, cfg.dueling, cfg.stream,
                       seed=seed, dyadic=dyadic)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("ddqn", [False, True], ids=["dqn", "ddqn"])
def test_c1_200_steps_teacher_forced(b, ddqn, precision):
    # BASELINE configs[0]: capacity 1000, D=27, 8 actions, B=32, 2x64 MLP, burn-in 100,
    # 200 executed train steps; 7 adds per iteration (the ring wraps in iteration 143);
    # target sync every 50 steps.  BF16 (reading Q33): one bf16 product per tensor-core
    # product, the north star's 2e-2 per step and for the 200-step drift
    tol = 1e-5 if precision == "fp32" else 2e-2
    cfg = _cfg(b, dueling=False, hidden=(64, 64), double_dqn=ddqn, sync_period=50, max_batch=32,
               precision=precision)
    p0 = _params(cfg)
    rp = b.Replay(1000, 27, burn_in=100, seed=2)
    dqn = b.DQN(cfg, p0)
    orc = oracle.Ring(1000, 27)
    e = experiences(214 * 7, seed=1)
    stats = {}
    ln = oracle.Learner(oracle_net(cfg), p0, gamma=f32(cfg.gamma), kappa=f32(cfg.huber_kappa),
                        lr=f32(cfg.lr), double_dqn=ddqn, burn_in=100, sync_period=50, seed=2)
    free_ring = oracle.Ring(1000, 27)
    executed = 0
    for it in range(1, 215):
        part = {k: v[(it - 1) * 7:it * 7] for k, v in e.items()}
        rp.add(**part)
        orc.add(**part)
        free_ring.add(**part)
        out = step_and_compare(b, cfg, dqn, rp, orc, 32, seed=2, burn_in=100, stats=stats, tol=tol)
        ln.step(free_ring, 32)
        if out is None:
            assert it <= 14
            continue
        executed += 1
        t = executed
        tgt = dqn.get_params(b.RPL_TARGET)
        if t % 50 == 0:
            assert np.array_equal(tgt, dqn.get_params(b.RPL_ONLINE))   # P:88 sync
        else:
            assert np.array_equal(tgt, out["target_before"])            # frozen
    assert executed == 200 and dqn.steps == 200
    # free-running drift of the fp32 device learner vs the fp64-arithmetic oracle learner
    drift = normwise(dqn.get_params(b.RPL_ONLINE), ln.online, 1e-3 if precision == "fp32" else 2e-2,
                     "200-step drift")
    print(f"\nC1 {'DDQN' if ddqn else 'DQN'} {precision}: 200 steps, mask flips replayed {stats['mask_flips']},"
          f" free-running drift {drift:.2e}")
    assert dqn.check() == b.RPL_OK


@pytest.mark.parametrize("ddqn", [False, True], ids=["dqn", "ddqn"])
def test_paper_dueling_1m_ring_b128(b, ddqn):
    # BASELINE configs[1]/[2]: 1,000,000-slot ring, 27-float states, batch 128, the paper's
    # dueling net (27 -> 128 -> V 512 / A 512 -> 1 + 8); sampled steps at full size
    cfg = _cfg(b, double_dqn=ddqn, lr=1e-3, max_batch=128, sync_period=2)
    rp = b.Replay(1_000_000, 27, seed=2)
    orc = oracle.Ring(1_000_000, 27)
    e = experiences(1_000_000, seed=1)
    rp.add_many(e)
    orc.add_many(e)
    dqn = b.DQN(cfg, _params(cfg))
    for _ in range(4):
        step_and_compare(b, cfg, dqn, rp, orc, 128, seed=2)
    assert np.array_equal(dqn.get_params(b.RPL_TARGET), dqn.get_params(b.RPL_ONLINE))


@pytest.mark.parametrize("batch", [1, 3, 33, 257, 1000, 4096])
def test_batch_sweep_ddqn(b, batch):
    # BASELINE configs[2]: Double DQN batch sweep 32..4096 plus ragged edge sizes
    cfg = _cfg(b, double_dqn=True, max_batch=4096)
    rp = b.Replay(50_000, 27, seed=5, rank=1)
    orc = oracle.Ring(50_000, 27)
    e = experiences(60_000, seed=6, done_prob=0.1)
    rp.add_many(e)
    orc.add_many(e)
    dqn = b.DQN(cfg, _params(cfg, seed=7))
    step_and_compare(b, cfg, dqn, rp, orc, batch, seed=5, rank=1)


@pytest.mark.parametrize("net", [dict(dueling=False, hidden=(64, 64)),
                                 dict(dueling=False, hidden=(50, 33, 17)),
                                 dict(dueling=True, hidden=(48, 40), stream=72, n_actions=5),
                                 dict(dueling=True, hidden=(128,), stream=512, n_actions=31)],
                         ids=["2x64", "3layer-ragged", "dueling-small", "dueling-A31"])
@pytest.mark.parametrize("kappa", [1.0, math.inf, 0.01])
def test_other_nets_and_kappas(b, net, kappa):
    cfg = _cfg(b, huber_kappa=kappa, double_dqn=True, max_batch=300, **net)
    rp = b.Replay(5000, 27, seed=11)
    orc = oracle.Ring(5000, 27)
    e = experiences(5000, n_actions=cfg.n_actions, seed=12)
    rp.add_many(e)
    orc.add_many(e)
    dqn = b.DQN(cfg, _params(cfg, seed=13))
    for batch in (300, 77):
        step_and_compare(b, cfg, dqn, rp, orc, batch, seed=11)


@pytest.mark.parametrize("dueling", [False, True])
def test_exact_input_mode_bitwise(b, dueling):
    # dyadic states/weights/rewards and gamma = 0.5: every forward activation, Q, argmax and
    # y (hence delta) is exact in fp32, so GPU == oracle bit for bit; the loss
    # (delta^2 needs > 24 bits) and gradients are checked at the FP32 tolerance
    cfg = _cfg(b, dueling=dueling, hidden=(128,) if dueling else (64, 64), gamma=0.5,
               double_dqn=True, max_batch=128)
    rp = b.Replay(4096, 27, seed=21)
    orc = oracle.Ring(4096, 27)
    e = experiences(4096, seed=22, dyadic=True)
    rp.add_many(e)
    orc.add_many(e)
    dqn = b.DQN(cfg, _params(cfg, seed=23, dyadic=True))
    dqn.set_params(_params(cfg, seed=24, dyadic=True), b.RPL_TARGET)
    step_and_compare(b, cfg, dqn, rp, orc, 128, seed=21, exact=True)


def test_burn_in_and_determinism_and_zero_h2d(b):
    cfg = _cfg(b, max_batch=64, sync_period=3)
    p0 = _params(cfg)
    runs = []
    for rep in range(2):
        rp = b.Replay(1000, 27, burn_in=200, seed=31)
        dqn = b.DQN(cfg, p0)
        e = experiences(600, seed=32)
        rp.add(**{k: v[:150] for k, v in e.items()})
        # during burn-in nothing is enqueued and no counter advances
        assert dqn.train_step(rp, 64) == b.RPL_NOT_READY
        assert rp.state()["events"] == 0 and dqn.steps == 0
        assert np.array_equal(dqn.get_params(b.RPL_ONLINE), p0)
        rp.add(**{k: v[150:] for k, v in e.items()})
        h2d = rp.state()["h2d_bytes"]
        for _ in range(10):
            assert dqn.train_step(rp, 64) == b.RPL_OK
        # a train step copies nothing from the host
        assert rp.state()["h2d_bytes"] == h2d == 600 * (8 * 27 + 9)
        runs.append(dqn.get_params(b.RPL_ONLINE).tobytes() + dqn.get_params(b.RPL_TARGET).tobytes())
    assert runs[0] == runs[1]   # same seeds -> byte-identical parameters


def test_nonfinite_loss_skips_update(b):
    import torch
    cfg = _cfg(b, max_batch=64, sync_period=1)
    rp = b.Replay(100, 27, seed=41)
    e = experiences(100, seed=42)
    e["r"][:] = np.nan
    rp.add(**e)
    dqn = b.DQN(cfg, _params(cfg))
    p_before = dqn.get_params(b.RPL_ONLINE)
    t_before = dqn.get_params(b.RPL_TARGET)
    loss = torch.zeros(1, device="cuda")
    assert dqn.train_step(rp, 64, loss) == b.RPL_OK
    assert dqn.check() == b.RPL_ENUMERIC
    assert np.isnan(loss.item())
    assert np.array_equal(dqn.get_params(b.RPL_ONLINE), p_before)
    assert np.array_equal(dqn.get_params(b.RPL_TARGET), t_before)


@pytest.mark.parametrize("path", ["fast", "generic"])
def test_action_outside_the_action_set_skips_update(b, path, monkeypatch):
    # the oracle rejects a batch holding an action outside [0, A) (test_oracle_dqn.py); the
    # device cannot return an argument error mid-stream, so the step skips its update and the
    # sticky ECORRUPT reports it
    if path == "generic":
        monkeypatch.setenv("RPL_PATH", "generic")
    import torch
    cfg = _cfg(b, max_batch=64, sync_period=1)
    rp = b.Replay(100, 27, seed=43)
    e = experiences(100, seed=44)
    e["a"][:] = 8   # A = 8
    rp.add(**e)
    dqn = b.DQN(cfg, _params(cfg))
    p_before = dqn.get_params(b.RPL_ONLINE)
    loss = torch.zeros(1, device="cuda")
    assert dqn.train_step(rp, 64, loss) == b.RPL_OK
    assert dqn.check() == b.RPL_ECORRUPT
    assert not np.isfinite(loss.item())
    assert np.array_equal(dqn.get_params(b.RPL_ONLINE), p_before)


def test_explicit_sync_target_and_set_get(b):
    cfg = _cfg(b, max_batch=32)
    rp = b.Replay(500, 27, seed=51)
    rp.add(**experiences(500, seed=52))
    dqn = b.DQN(cfg, _params(cfg))
    for _ in range(3):
        dqn.train_step(rp, 32)
    assert not np.array_equal(dqn.get_params(b.RPL_TARGET), dqn.get_params(b.RPL_ONLINE))
    dqn.sync_target()
    assert np.array_equal(dqn.get_params(b.RPL_TARGET), dqn.get_params(b.RPL_ONLINE))
    with pytest.raises(b.RplError):
        dqn.train_step(rp, 33)   # > max_batch
    with pytest.raises(b.RplError):
        dqn.set_params(np.zeros(5, np.float32))


@pytest.mark.parametrize("mode", ["host", "device_defer", "mixed"])
def test_deferred_insert_read_through(b, mode):
    # replay_add's ring write deferred into the train step's first kernel (include/
    # ingpu_replay.h, replay_add): with a 64-slot ring, 8 adds per step and batch 128 almost
    # every step samples slots of the pending insert, which are read from its sources; the
    # pending range wraps the ring end every 8th step.  Sampled batch bit-exact, the step
    # within tolerance, and the ring contents exact afterwards.
    import torch
    cfg = _cfg(b, max_batch=128, double_dqn=True, sync_period=3)
    C = 64
    rp = b.Replay(C, 27, burn_in=16, seed=5)
    orc = oracle.Ring(C, 27)
    dqn = b.DQN(cfg, _params(cfg))
    e = experiences(8 * 40, seed=11)
    dev = {k: torch.from_numpy(v).cuda() for k, v in e.items()}
    hits = 0
    for it in range(40):
        sl = slice(8 * it, 8 * it + 8)
        if mode == "device_defer" or (mode == "mixed" and it % 2):
            rp.add(**{k: v[sl] for k, v in dev.items()}, defer=True)
        else:
            rp.add(**{k: v[sl] for k, v in e.items()})
        orc.add(**{k: v[sl] for k, v in e.items()})
        if mode == "mixed" and it % 5 == 4 and it > 2:
            # any other call on the replay writes the pending insert first
            g = rp.sample(16)
            rc, o = orc.sample(16, 5, 0, 16)
            assert rc == oracle.OK
            for k in ("idx", "s", "s_next", "a", "r", "done"):
                assert np.array_equal(g[k].cpu().numpy(), o[k]), k
        st = rp.state()
        cur = st["cursor"]
        out = step_and_compare(b, cfg, dqn, rp, orc, 128, seed=5, burn_in=16)
        if out is not None:
            idx = dqn.debug(b.RPL_DBG_IDX, 128).astype(np.int64)
            hits += int(((idx - (cur - 8)) % C < 8).sum())
    assert hits > 300   # ~16 of 128 rows per step
    idx = torch.arange(C, dtype=torch.int32, device="cuda")
    g = rp.gather(idx)
    o = orc.gather(np.arange(C, dtype=np.int32))
    for k in ("s", "s_next", "a", "r", "done"):
        assert np.array_equal(g[k].cpu().numpy(), o[k]), k
    assert rp.check() == b.RPL_OK and dqn.check() == b.RPL_OK


def test_deferred_device_insert_corrupt_done(b):
    # a device-sourced done > 1 is stored as 1 and raises the replay's sticky ECORRUPT,
    # also when the deferred write happens inside the train step
    import torch
    cfg = _cfg(b, max_batch=32)
    rp = b.Replay(50, 27, seed=61)
    e = experiences(48, seed=62)
    rp.add(**e)
    dqn = b.DQN(cfg, _params(cfg))
    bad = {k: torch.from_numpy(v[:2].copy()).cuda() for k, v in e.items()}
    bad["done"][0] = 7
    rp.add(**bad, defer=True)
    assert dqn.train_step(rp, 32) == b.RPL_OK
    assert dqn.check() == b.RPL_OK
    assert rp.check() == b.RPL_ECORRUPT
    g = rp.gather(torch.tensor([48, 49], dtype=torch.int32, device="cuda"))
    assert g["done"].cpu().numpy().tolist() == [1, int(e["done"][1])]


@pytest.mark.parametrize("batch", [128, 640])
def test_loss_destination_device_and_pinned_host(b, batch):
    # a pinned-host loss destination takes the step graph with the loss side branch
    # (loss_out_kernel), a device one the graph whose K4 writes it: alternating the two on one
    # learner must give, step for step, the loss of a learner that always writes to the device
    import torch
    cfg = _cfg(b, double_dqn=True, sync_period=3, max_batch=batch)
    p0 = _params(cfg, seed=23)
    e = experiences(3000, seed=24)
    losses = []
    for alternate in (False, True):
        rp = b.Replay(3000, 27, seed=25)
        rp.add(**e)
        dqn = b.DQN(cfg, p0)
        dev = torch.zeros(1, device="cuda")
        host = torch.zeros(8, dtype=torch.float32, pin_memory=True)
        out = []
        for i in range(8):
            dst = host[i:i + 1] if (alternate and i % 2 == 1) else dev
            assert dqn.train_step(rp, batch, dst) == b.RPL_OK
            torch.cuda.synchronize()
            out.append(float(dst.cpu()[0]) if dst is dev else float(dst[0]))
        assert dqn.check() == b.RPL_OK
        losses.append(out)
    assert losses[0] == losses[1]
    assert all(np.isfinite(losses[0])) and all(v > 0 for v in losses[0])
