"""Pins for the oracle's decision-replay inputs and for O6, the data-parallel mean (CPU only).

`oracle_dqn_loss_grad(mask_override, argmax_override)` re-evaluates the P:90 update under
decisions taken by the GPU (reading Q25 "decision replay": a ReLU unit whose pre-activation is
within rounding of 0, a Double-DQN argmax whose top two online Q are within rounding).  These
tests pin that path against things other than the oracle itself:

* overrides equal to the natural decisions are bit-identical to no override;
* forcing a unit with z = 0 exactly (a dyadic net built for it) on, or any unit to an arbitrary
  state, equals an independent torch float64 autograd of the same graph with h = z * m on the
  online forward of s (the only forward whose masks the GPU exports);
* on an exact Double-DQN tie (lowest index by Q19) `argmax_override = 1` gives
  y = r + gamma (1 - d) Q_t(s', 1).

O6 (`oracle_dp_mean_sgd`, "the model synchronized every train step", readings Q22/Q23)
is pinned by: world 1 = plain SGD; the rank-order sum of dyadic gradients against exact
integer arithmetic; equal per-rank batches -> the mean of the per-rank batch-mean gradients
equals the gradient of the concatenated global batch (the identity Q23 rests on).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from inputs import experiences, init_params, layer_shapes


def _unpack(net, theta):
    out, o = [], 0
    for (r, c) in layer_shapes(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream):
        out.append((theta[o:o + r * c].reshape(r, c), theta[o + r * c:o + r * c + r]))
        o += r * c + r
    return out


def _q(net, theta, x, mask=None):
    """Q(x) in torch float64; mask [B x H] (hidden-unit space: shared layers, then the 2S
    stream units [V | A]) replaces ReLU by h = z * m."""
    layers = _unpack(net, theta)
    h, off = x, 0

    def act(z):
        nonlocal off
        n = z.shape[1]
        if mask is None:
            out = torch.relu(z)
        else:
            out = z * mask[:, off:off + n]
        off += n
        return out

    for W, b in layers[:len(net.hidden)]:
        h = act(torch.nn.functional.linear(h, W, b))
    if not net.dueling:
        W, b = layers[-1]
        return torch.nn.functional.linear(h, W, b)
    S = net.stream
    hs = act(torch.nn.functional.linear(h, *layers[-2]))
    Whd, bhd = layers[-1]
    V = hs[:, :S] @ Whd[0] + bhd[0]
    Aa = hs[:, S:] @ Whd[1:].T + bhd[1:]
    return V[:, None] + Aa - Aa.mean(dim=1, keepdim=True)


def _torch_eval(net, online, target, e, gamma, kappa, ddqn, mask=None, a_star=None):
    th = torch.tensor(online, dtype=torch.float64, requires_grad=True)
    tg = torch.tensor(target, dtype=torch.float64)
    s = torch.tensor(e["s"], dtype=torch.float64)
    s2 = torch.tensor(e["s_next"], dtype=torch.float64)
    a = torch.tensor(e["a"], dtype=torch.int64)
    r = torch.tensor(e["r"], dtype=torch.float64)
    d = torch.tensor(e["done"], dtype=torch.float64)
    m = None if mask is None else torch.tensor(mask, dtype=torch.float64)
    with torch.no_grad():
        qt = _q(net, tg, s2)
        if ddqn:
            sel = (_q(net, th, s2).argmax(dim=1) if a_star is None
                   else torch.tensor(a_star, dtype=torch.int64))
            boot = qt.gather(1, sel[:, None])[:, 0]
        else:
            boot = qt.max(dim=1).values
        y = r + gamma * (1 - d) * boot
    qs = _q(net, th, s, m).gather(1, a[:, None])[:, 0]
    if math.isinf(kappa):
        loss = (0.5 * (qs - y) ** 2).mean()
    else:
        loss = torch.nn.functional.huber_loss(qs, y, reduction="mean", delta=kappa)
    loss.backward()
    return loss.item(), th.grad.numpy().copy(), y.numpy()


NETS = [
    oracle.Net(state_dim=27, n_actions=8, dueling=False, hidden=(64, 64)),
    oracle.Net(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512),
    oracle.Net(state_dim=5, n_actions=3, dueling=True, hidden=(6, 7), stream=11),
]
IDS = ["2x64", "paper-dueling", "deep-dueling"]


@pytest.mark.parametrize("net", NETS, ids=IDS)
@pytest.mark.parametrize("ddqn", [False, True])
def test_natural_overrides_are_bit_identical_to_none(net, ddqn):
    th = init_params(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream, seed=91)
    tg = init_params(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream, seed=92)
    e = experiences(48, net.state_dim, net.n_actions, seed=93, done_prob=0.2)
    base = oracle.dqn_loss_grad(net, th, tg, e, 0.99, 1.0, ddqn)
    rep = oracle.dqn_loss_grad(net, th, tg, e, 0.99, 1.0, ddqn, mask_override=base["on"],
                               argmax_override=base["a_star"] if ddqn else None)
    assert rep["loss"] == base["loss"]
    for k in ("grad", "q_s", "q_next_target", "y", "z", "on"):
        assert np.array_equal(rep[k], base[k]), k
    assert 0 < base["on"].mean() < 1   # the natural masks exercise both decisions


def _zero_unit_net():
    """Plain 2-layer net (D=4, hidden (6, 5), A=3) with dyadic weights, built so that hidden
    unit 2 of layer 0 has z = 0 exactly for sample 0 and the layer above depends on it."""
    net = oracle.Net(state_dim=4, n_actions=3, dueling=False, hidden=(6, 5))
    th = init_params(4, 3, (6, 5), False, seed=94, dyadic=True).astype(np.float64)
    e = experiences(4, 4, 3, seed=95, dyadic=True, done_prob=0.0)
    W0 = th[:24].reshape(6, 4)
    # z[0, 2] = W0[2] . s0 + b0[2] = 0: choose the bias as minus the dot product (dyadic, exact)
    th[24 + 2] = -float(W0[2] @ e["s"][0].astype(np.float64))
    # unit 2 feeds layer 1 with nonzero weights so forcing it changes the gradient
    W1 = th[30:60].reshape(5, 6)
    W1[:, 2] = 0.25
    th[30:60] = W1.ravel()
    return net, th, e


def test_forcing_a_zero_preactivation_unit_on_matches_torch():
    net, th, e = _zero_unit_net()
    base = oracle.dqn_loss_grad(net, th, th, e, 0.5, 1.0, False)
    assert base["z"][0, 2] == 0.0 and base["on"][0, 2] == 0   # ReLU'(0) = 0 (Q13)
    forced = base["on"].copy()
    forced[0, 2] = 1
    rep = oracle.dqn_loss_grad(net, th, th, e, 0.5, 1.0, False, mask_override=forced)
    # same forward (h = z = 0 either way), different gradient: d z flows through unit 2
    assert np.array_equal(rep["q_s"], base["q_s"]) and rep["loss"] == base["loss"]
    assert not np.array_equal(rep["grad"], base["grad"])
    tl, tgrad, _ = _torch_eval(net, th, th, e, 0.5, 1.0, False, mask=forced.astype(np.float64))
    assert rep["loss"] == pytest.approx(tl, rel=1e-14, abs=0)
    assert np.max(np.abs(rep["grad"] - tgrad)) <= 1e-14 * np.max(np.abs(tgrad))
    # and the natural mask matches torch's ReLU (ReLU'(0) = 0 in torch too)
    _, tnat, _ = _torch_eval(net, th, th, e, 0.5, 1.0, False)
    assert np.max(np.abs(base["grad"] - tnat)) <= 1e-14 * np.max(np.abs(tnat))


@pytest.mark.parametrize("net", NETS, ids=IDS)
@pytest.mark.parametrize("ddqn", [False, True])
@pytest.mark.parametrize("kappa", [1.0, math.inf])
def test_arbitrary_mask_override_matches_torch(net, ddqn, kappa):
    # any replayed mask (here: 5% of the natural decisions flipped) is the graph with h = z * m
    # on the online forward of s; the s' forwards keep their natural ReLU
    th = init_params(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream, seed=96)
    tg = init_params(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream, seed=97)
    e = experiences(24, net.state_dim, net.n_actions, seed=98, done_prob=0.25)
    base = oracle.dqn_loss_grad(net, th, tg, e, 0.99, kappa, ddqn)
    flip = np.random.default_rng(99).random(base["on"].shape) < 0.05
    mask = base["on"] ^ flip.astype(np.uint8)
    rep = oracle.dqn_loss_grad(net, th, tg, e, 0.99, kappa, ddqn, mask_override=mask)
    tl, tgrad, ty = _torch_eval(net, th.astype(np.float64), tg.astype(np.float64), e, 0.99, kappa,
                                ddqn, mask=mask.astype(np.float64))
    assert rep["loss"] == pytest.approx(tl, rel=1e-12, abs=1e-15)
    assert np.max(np.abs(rep["grad"] - tgrad)) <= 1e-12 * max(1.0, np.max(np.abs(tgrad)))
    assert np.allclose(rep["y"], ty, rtol=1e-13, atol=1e-15)
    assert not np.array_equal(rep["grad"], base["grad"])
    assert np.array_equal(rep["on"], mask)   # the exported decisions are the replayed ones


def _const_head_net(A, q_values):
    """plain net whose Q(s, .) = q_values for every s (head weights 0)"""
    net = oracle.Net(state_dim=2, n_actions=A, dueling=False, hidden=(2,))
    theta = np.concatenate([np.eye(2).ravel(), np.zeros(2), np.zeros(2 * A),
                            np.asarray(q_values, np.float64)])
    return net, theta


def test_argmax_override_on_an_exact_ddqn_tie():
    # online Q(s', .) = [1, 1] (exact tie -> action 0 by Q19); target Q(s', .) = [0.5, 1.5]
    net, online = _const_head_net(2, [1.0, 1.0])
    _, target = _const_head_net(2, [0.5, 1.5])
    e = dict(s=np.zeros((3, 2), np.float32), a=np.array([0, 1, 0], np.int32),
             r=np.array([1.0, -0.25, 0.25], np.float32), s_next=np.ones((3, 2), np.float32),
             done=np.array([0, 0, 1], np.uint8))
    gamma = 0.75
    nat = oracle.dqn_loss_grad(net, online, target, e, gamma, 1.0, True)
    assert nat["a_star"].tolist() == [0, 0, 0]
    assert np.array_equal(nat["y"], e["r"] + gamma * (1 - e["done"]) * 0.5)
    rep = oracle.dqn_loss_grad(net, online, target, e, gamma, 1.0, True,
                               argmax_override=np.ones(3, np.int32))
    assert rep["a_star"].tolist() == [1, 1, 1]
    # y = r + gamma (1 - d) Q_t(s', 1); the terminal sample keeps y = r
    assert np.array_equal(rep["y"], e["r"].astype(np.float64) + gamma * (1 - e["done"]) * 1.5)
    tl, tgrad, ty = _torch_eval(net, online, target, e, gamma, 1.0, True,
                                a_star=np.ones(3, np.int64))
    assert np.array_equal(rep["y"], ty)
    assert rep["loss"] == pytest.approx(tl, rel=1e-15, abs=0)
    assert np.max(np.abs(rep["grad"] - tgrad)) <= 1e-15 * max(1.0, np.max(np.abs(tgrad)))
    # the override changes only y (the selection is stop-gradient)
    assert rep["loss"] != nat["loss"]


# ------------------------------------------------------------------------------------
# O6: data-parallel mean + SGD
# ------------------------------------------------------------------------------------
def test_dp_mean_world1_is_plain_sgd():
    w = np.random.default_rng(1).standard_normal(1000)
    g = np.random.default_rng(2).standard_normal(1000)
    w1, mean = oracle.dp_mean_sgd(w, [g], 1e-3)
    assert np.array_equal(w1, oracle.sgd(w, g, 1e-3)) and np.array_equal(mean, g)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_dp_mean_rank_order_sum_exact_on_dyadics(world):
    # dyadic gradients with small numerators: every partial sum and the division by a power of
    # two are exact, so the mean equals the integer sum / N computed with Python integers
    rng = np.random.default_rng(world)
    num = rng.integers(-1000, 1000, size=(world, 257))
    grads = [num[r] / 64.0 for r in range(world)]
    w = rng.integers(-64, 64, size=257) / 8.0
    lr = 0.5
    w1, mean = oracle.dp_mean_sgd(w, grads, lr)
    tot = num.sum(axis=0)
    if world & (world - 1) == 0:
        assert np.array_equal(mean, tot / (64.0 * world))
        assert np.array_equal(w1, w - lr * (tot / (64.0 * world)))
    else:
        assert np.allclose(mean, tot / (64.0 * world), rtol=1e-15, atol=0)
    # identical gradients on every rank: the mean is that gradient (the world-N identical-shard
    # learner equals the single learner)
    w2, mean2 = oracle.dp_mean_sgd(w, [grads[0]] * world, lr)
    assert np.array_equal(mean2, grads[0]) if world & (world - 1) == 0 else \
        np.allclose(mean2, grads[0], rtol=1e-15, atol=0)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("ddqn", [False, True])
def test_dp_mean_of_shard_gradients_equals_global_batch_gradient(world, ddqn):
    # Q23: for equal per-rank B, (1/N) sum_r (1/B) sum_{i in r} dL_i = (1/(NB)) sum_i dL_i --
    # the gradient of the concatenated batch of N*B samples (an identity of the mean)
    net = oracle.Net(27, 8, True, (128,), 512)
    th = init_params(seed=101)
    tg = init_params(seed=102)
    B = 16
    shards = [experiences(B, seed=103, rank=r, done_prob=0.1) for r in range(world)]
    grads, losses = [], []
    for e in shards:
        o = oracle.dqn_loss_grad(net, th, tg, e, 0.99, 1.0, ddqn)
        grads.append(o["grad"]); losses.append(o["loss"])
    glob = {k: np.concatenate([e[k] for e in shards]) for k in shards[0]}
    og = oracle.dqn_loss_grad(net, th, tg, glob, 0.99, 1.0, ddqn)
    lr = 1e-3
    w1, mean = oracle.dp_mean_sgd(th, grads, lr)
    scale = np.max(np.abs(og["grad"]))
    assert np.max(np.abs(mean - og["grad"])) <= 1e-13 * scale
    assert np.mean(losses) == pytest.approx(og["loss"], rel=1e-13)
    assert np.max(np.abs(w1 - oracle.sgd(th, og["grad"], lr))) <= 1e-15


# ------------------------------------------------------------------------------------
# tests/golden/paper_worked_examples.txt: every value there is checked here
# ------------------------------------------------------------------------------------
def _golden():
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", "paper_worked_examples.txt")
    out = {}
    for line in open(p):
        if line.startswith("#") or not line.strip():
            continue
        name, val, _cite = [x.strip() for x in line.split("|", 2)]
        out[name] = val
    return out


def test_golden_paper_worked_examples():
    g = _golden()
    assert set(g) == {"row_width_D27", "duplicate_rate_B32_n1e6", "pack_D2", "select_q",
                      "td_target", "dueling_combine", "target_sync_period"}
    # the packed row of a 27-float state is 57 floats
    assert oracle.Ring(4, 27).rows().shape[1] == int(g["row_width_D27"])
    # duplicate probability at B = 32 from 1M slots, birthday product, rounds to 0.05 %
    p = 1.0 - np.prod([1.0 - i / 1e6 for i in range(32)])
    assert round(p, 4) == float(g["duplicate_rate_B32_n1e6"])
    # S:52 pack example in the paper's layout
    ring = oracle.Ring(2, 2)
    ring.add(s=np.array([[1, 2]], np.float32), a=np.array([3], np.int32),
             r=np.array([0.5], np.float32), s_next=np.array([[4, 5]], np.float32),
             done=np.array([1], np.uint8))
    assert ring.rows()[0].tolist() == [float(x) for x in g["pack_D2"].split(",")]
    # S:285 select, with (a..f) = (1..6)
    net = oracle.Net(state_dim=2, n_actions=3, dueling=False, hidden=(2,))
    vals = dict(a=1.0, b=2.0, c=3.0, d=4.0, e=5.0, f=6.0)
    Wo = np.array([[vals["a"], vals["d"]], [vals["b"], vals["e"]], [vals["c"], vals["f"]]])
    th = np.concatenate([np.eye(2).ravel(), np.zeros(2), Wo.ravel(), np.zeros(3)])
    bt = dict(s=np.array([[1, 0], [0, 1]], np.float32), a=np.array([2, 0], np.int32),
              r=np.zeros(2, np.float32), s_next=np.zeros((2, 2), np.float32),
              done=np.zeros(2, np.uint8))
    out = oracle.dqn_loss_grad(net, th, th, bt, 0.0, math.inf, False)
    sel = [out["q_s"][i, bt["a"][i]] for i in range(2)]
    assert sel == [vals[x] for x in g["select_q"].split(",")]
    # S:296 TD target
    net2, tgt = _const_head_net(2, [0.5, 1.5])
    b2 = dict(s=np.zeros((1, 2), np.float32), a=np.zeros(1, np.int32),
              r=np.ones(1, np.float32), s_next=np.zeros((1, 2), np.float32),
              done=np.zeros(1, np.uint8))
    assert oracle.dqn_loss_grad(net2, tgt, tgt, b2, 0.99, 1.0, False)["y"][0] == \
        pytest.approx(float(g["td_target"]), abs=1e-15)
    # S:276 dueling combine
    S, A = 4, 3
    netd = oracle.Net(state_dim=2, n_actions=A, dueling=True, hidden=(2,), stream=S)
    thd = np.concatenate([np.eye(2).ravel(), np.zeros(2), np.zeros(2 * S * 2), np.zeros(2 * S),
                          np.zeros((1 + A) * S), [1.0, 1.0, 2.0, 3.0]])
    bd = dict(s=np.ones((1, 2), np.float32), a=np.zeros(1, np.int32), r=np.zeros(1, np.float32),
              s_next=np.ones((1, 2), np.float32), done=np.zeros(1, np.uint8))
    q = oracle.dqn_loss_grad(netd, thd, thd, bd, 0.5, 1.0, False)["q_s"][0]
    assert q.tolist() == [float(x) for x in g["dueling_combine"].split(",")]
    # P:88 target sync period: the learner syncs after every period-th step
    per = int(g["target_sync_period"])
    assert per == 10000
    ln = oracle.Learner(net2, tgt, sync_period=per)
    assert ln._l.sync_period == per
