"""Pins for the oracle's Q-network, TD target, Huber loss, gradient, SGD and target sync.

Pinned against: the paper's equations evaluated on hand-built nets,
SPEC worked examples, central finite differences (fp64), an independent torch float64
autograd implementation of the same graph (library-routine pin), and invariants of the
dueling combine.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from inputs import experiences, init_params, layer_shapes

INF = math.inf


def _blob(parts):
    return np.concatenate([np.asarray(p, np.float64).ravel() for p in parts])


# ------------------------------------------------------------------------------------
# worked examples on hand-built nets
# ------------------------------------------------------------------------------------
def test_select_q_enumerate_mask_example():
    # S:285 / P:79-81: q = [[a,b,c],[d,e,f]], actions [2,0] -> [c, d]
    a_, b_, c_, d_, e_, f_ = 0.5, -1.25, 2.0, 3.5, 0.25, -0.75
    net = oracle.Net(state_dim=2, n_actions=3, dueling=False, hidden=(2,))
    W1, b1 = np.eye(2), np.zeros(2)          # h = ReLU(s) = s for s >= 0
    Wo = np.array([[a_, d_], [b_, e_], [c_, f_]])  # Q(s1=[1,0]) = [a,b,c]; Q(s2=[0,1]) = [d,e,f]
    theta = _blob([W1, b1, Wo, np.zeros(3)])
    batch = dict(s=np.array([[1, 0], [0, 1]], np.float32), a=np.array([2, 0]),
                 r=np.zeros(2, np.float32), s_next=np.zeros((2, 2), np.float32),
                 done=np.zeros(2, np.uint8))
    out = oracle.dqn_loss_grad(net, theta, theta, batch, gamma=0.0, kappa=INF, double_dqn=False)
    assert np.allclose(out["q_s"], [[a_, b_, c_], [d_, e_, f_]], atol=0, rtol=0)
    # gamma = 0 -> y = r = 0, delta_i = q[i, a_i] = [c, d]; L = mean(1/2 delta^2)
    assert out["loss"] == pytest.approx(0.5 * (c_ * c_ + d_ * d_) / 2, abs=0)


def _const_head_net(A, q_values):
    """plain net whose Q(s, .) = q_values for every s (head weights 0)"""
    net = oracle.Net(state_dim=2, n_actions=A, dueling=False, hidden=(2,))
    theta = _blob([np.eye(2), np.zeros(2), np.zeros((A, 2)), np.asarray(q_values)])
    return net, theta


def test_td_target_examples():
    # S:294-296 / P:90: r=1, gamma=0.99, next=[0.5,1.5], not terminal -> 2.485
    net, tgt = _const_head_net(2, [0.5, 1.5])
    batch = dict(s=np.zeros((3, 2), np.float32), a=np.zeros(3, np.int32),
                 r=np.array([1.0, 2.0, 1.0], np.float32), s_next=np.zeros((3, 2), np.float32),
                 done=np.array([0, 1, 0], np.uint8))
    out = oracle.dqn_loss_grad(net, tgt, tgt, batch, gamma=0.99, kappa=1.0, double_dqn=False)
    assert out["y"][0] == pytest.approx(2.485, abs=1e-15)
    assert out["y"][1] == 2.0  # terminal -> y = r regardless of next Q
    out0 = oracle.dqn_loss_grad(net, tgt, tgt, batch, gamma=0.0, kappa=1.0, double_dqn=False)
    assert np.array_equal(out0["y"], batch["r"].astype(np.float64))  # gamma = 0 -> y = r
    # DDQN: select with the online net, evaluate with the target (Q9)
    net_o, onl = _const_head_net(2, [9.0, -9.0])  # online prefers action 0
    outd = oracle.dqn_loss_grad(net, onl, tgt, batch, gamma=0.99, kappa=1.0, double_dqn=True)
    assert outd["a_star"].tolist() == [0, 0, 0]
    assert outd["y"][0] == pytest.approx(1 + 0.99 * 0.5, abs=1e-15)
    # ties -> lowest index (Q19)
    net_t, tie = _const_head_net(2, [1.0, 1.0])
    outt = oracle.dqn_loss_grad(net, tie, tgt, batch, gamma=0.99, kappa=1.0, double_dqn=True)
    assert outt["a_star"].tolist() == [0, 0, 0]


def test_dueling_combine_example_and_invariants():
    # S:276 / P:94: V = 1, A = [1,2,3] -> Q = [0,1,2]
    S, A = 4, 3
    net = oracle.Net(state_dim=2, n_actions=A, dueling=True, hidden=(2,), stream=S)
    theta = _blob([np.eye(2), np.zeros(2), np.zeros((2 * S, 2)), np.zeros(2 * S),
                   np.zeros((1 + A, S)), [1.0, 1.0, 2.0, 3.0]])
    batch = dict(s=np.ones((1, 2), np.float32), a=np.zeros(1, np.int32), r=np.zeros(1, np.float32),
                 s_next=np.ones((1, 2), np.float32), done=np.zeros(1, np.uint8))
    out = oracle.dqn_loss_grad(net, theta, theta, batch, gamma=0.5, kappa=1.0, double_dqn=False)
    assert out["q_s"][0].tolist() == [0.0, 1.0, 2.0]

    # random dueling net: (i) adding c to every A-head bias leaves Q unchanged;
    # (ii) adding c to the V bias shifts every Q by c; (iii) zero A head -> Q = V for all a,
    # so mean_a Q = V
    net = oracle.Net(state_dim=5, n_actions=6, dueling=True, hidden=(7,), stream=9)
    th = init_params(5, 6, (7,), True, 9, seed=4).astype(np.float64)
    e = experiences(16, 5, 6, seed=3)
    base = oracle.dqn_loss_grad(net, th, th, e, 0.9, 1.0, False)["q_s"]
    P = net.param_count
    hb = P - (1 + 6)  # start of b_hd = [b_V, b_A1..b_A6]
    th2 = th.copy(); th2[hb + 1:] += 0.375
    assert np.allclose(oracle.dqn_loss_grad(net, th2, th2, e, 0.9, 1.0, False)["q_s"], base,
                       rtol=0, atol=1e-12)
    th3 = th.copy(); th3[hb] += 0.375
    assert np.allclose(oracle.dqn_loss_grad(net, th3, th3, e, 0.9, 1.0, False)["q_s"], base + 0.375,
                       rtol=0, atol=1e-12)
    th4 = th.copy()
    hw = hb - (1 + 6) * 9   # start of W_hd
    th4[hw + 9:hb] = 0.0; th4[hb + 1:] = 0.0   # A head = 0
    q4 = oracle.dqn_loss_grad(net, th4, th4, e, 0.9, 1.0, False)["q_s"]
    assert np.allclose(q4, q4[:, :1], rtol=0, atol=0)


# ------------------------------------------------------------------------------------
# an independent torch float64 implementation of the same graph (library-routine pin)
# ------------------------------------------------------------------------------------
def _torch_loss(net, online, target, e, gamma, kappa, ddqn):
    shapes = layer_shapes(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream)

    def unpack(theta):
        out, o = [], 0
        for (r, c) in shapes:
            W = theta[o:o + r * c].reshape(r, c); o += r * c
            b = theta[o:o + r]; o += r
            out.append((W, b))
        return out

    def q(theta, x):
        layers = unpack(theta)
        h = x
        for W, b in layers[:len(net.hidden)]:
            h = torch.relu(torch.nn.functional.linear(h, W, b))
        if not net.dueling:
            W, b = layers[-1]
            return torch.nn.functional.linear(h, W, b)
        S = net.stream
        Wst, bst = layers[-2]
        hs = torch.relu(torch.nn.functional.linear(h, Wst, bst))
        hv, ha = hs[:, :S], hs[:, S:]
        Whd, bhd = layers[-1]
        V = hv @ Whd[0] + bhd[0]
        Aadv = ha @ Whd[1:].T + bhd[1:]
        return V[:, None] + Aadv - Aadv.mean(dim=1, keepdim=True)

    th = torch.tensor(online, dtype=torch.float64, requires_grad=True)
    tg = torch.tensor(target, dtype=torch.float64)
    s = torch.tensor(e["s"], dtype=torch.float64)
    s2 = torch.tensor(e["s_next"], dtype=torch.float64)
    a = torch.tensor(e["a"], dtype=torch.int64)
    r = torch.tensor(e["r"], dtype=torch.float64)
    d = torch.tensor(e["done"], dtype=torch.float64)
    with torch.no_grad():
        qt = q(tg, s2)
        if ddqn:
            boot = qt.gather(1, q(th, s2).argmax(dim=1, keepdim=True))[:, 0]
        else:
            boot = qt.max(dim=1).values
        y = r + gamma * (1 - d) * boot
    qs = q(th, s).gather(1, a[:, None])[:, 0]
    if math.isinf(kappa):
        loss = (0.5 * (qs - y) ** 2).mean()
    else:
        loss = torch.nn.functional.huber_loss(qs, y, reduction="mean", delta=kappa)
    loss.backward()
    return loss.item(), th.grad.numpy().copy()


NETS = [
    oracle.Net(state_dim=27, n_actions=8, dueling=False, hidden=(64, 64)),   # C1 net
    oracle.Net(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512),  # paper
    oracle.Net(state_dim=5, n_actions=3, dueling=True, hidden=(6, 7), stream=11),
    oracle.Net(state_dim=3, n_actions=2, dueling=False, hidden=(5, 4, 3)),
]


@pytest.mark.parametrize("net", NETS, ids=lambda n: f"D{n.state_dim}A{n.n_actions}h{n.hidden}d{int(n.dueling)}")
@pytest.mark.parametrize("ddqn", [False, True])
@pytest.mark.parametrize("kappa", [1.0, INF, 0.05])
def test_loss_and_grad_match_torch_autograd(net, ddqn, kappa):
    B = 32
    th = init_params(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream, seed=11)
    tg = init_params(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream, seed=12)
    e = experiences(B, net.state_dim, net.n_actions, seed=13, done_prob=0.25)
    out = oracle.dqn_loss_grad(net, th, tg, e, 0.99, kappa, ddqn)
    tl, tgrad = _torch_loss(net, th.astype(np.float64), tg.astype(np.float64), e, 0.99, kappa, ddqn)
    assert out["loss"] == pytest.approx(tl, rel=1e-12, abs=1e-15)
    assert np.max(np.abs(out["grad"] - tgrad)) <= 1e-12 * max(1.0, np.max(np.abs(tgrad)))
    assert np.any(out["grad"] != 0)


@pytest.mark.parametrize("net", [oracle.Net(3, 2, False, (4, 3)), oracle.Net(3, 2, True, (4,), 5)],
                         ids=["plain", "dueling"])
@pytest.mark.parametrize("ddqn", [False, True])
def test_grad_central_finite_differences(net, ddqn):
    # analytic gradient vs central differences, relative error < 1e-4 (fp64),
    # on every parameter block
    B = 6
    th = init_params(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream, seed=21,
                     bias_scale=0.3).astype(np.float64)
    tg = init_params(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream, seed=22,
                     bias_scale=0.3).astype(np.float64)
    e = experiences(B, net.state_dim, net.n_actions, seed=23, done_prob=0.3)
    g = oracle.dqn_loss_grad(net, th, tg, e, 0.9, 0.5, ddqn)["grad"]
    h = 1e-6
    fd = np.zeros_like(th)
    for i in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[i] += h; tm[i] -= h
        # the target net is frozen: only the online copy is perturbed
        fp = oracle.dqn_loss_grad(net, tp, tg, e, 0.9, 0.5, ddqn)["loss"]
        fm = oracle.dqn_loss_grad(net, tm, tg, e, 0.9, 0.5, ddqn)["loss"]
        fd[i] = (fp - fm) / (2 * h)
    o = 0
    for (r, c) in layer_shapes(net.state_dim, net.n_actions, net.hidden, net.dueling, net.stream):
        for n in (r * c, r):
            blk = slice(o, o + n)
            den = max(np.max(np.abs(fd[blk])), 1e-8)
            assert np.max(np.abs(g[blk] - fd[blk])) / den < 1e-4
            o += n
    assert o == th.size


def test_paper_update_rule_kappa_inf_batch1():
    # w <- w + alpha (r + gamma max_a' Q(s',a') - Q(s,a)) grad_w Q(s,a).  With kappa = inf
    # (1/2 delta^2) and B = 1 one SGD step must equal it; grad_w Q from torch autograd.
    net = oracle.Net(27, 8, True, (128,), 512)
    th = init_params(seed=31).astype(np.float64)
    tg = init_params(seed=32).astype(np.float64)
    e = experiences(1, seed=33, done_prob=0.0)
    out = oracle.dqn_loss_grad(net, th, tg, e, 0.99, INF, False)
    alpha = 1e-3
    w_new = oracle.sgd(th, out["grad"], alpha)
    # independent: grad of Q(s, a) alone (not of the loss)
    shapes = layer_shapes(27, 8, (128,), True, 512)
    t = torch.tensor(th, requires_grad=True)
    o, L = 0, []
    for (r, c) in shapes:
        L.append((t[o:o + r * c].reshape(r, c), t[o + r * c:o + r * c + r])); o += r * c + r
    x = torch.tensor(e["s"], dtype=torch.float64)
    h1 = torch.relu(torch.nn.functional.linear(x, *L[0]))
    hs = torch.relu(torch.nn.functional.linear(h1, *L[1]))
    Whd, bhd = L[2]
    V = hs[:, :512] @ Whd[0] + bhd[0]
    Aa = hs[:, 512:] @ Whd[1:].T + bhd[1:]
    Q = V[:, None] + Aa - Aa.mean(1, keepdim=True)
    Q[0, int(e["a"][0])].backward()
    y = out["y"][0]
    qsa = out["q_s"][0, e["a"][0]]
    expect = th + alpha * (y - qsa) * t.grad.numpy()
    assert np.max(np.abs(w_new - expect)) < 1e-15 * max(1, np.max(np.abs(th))) + 1e-16


def test_sgd_alpha_zero_and_small_step_reduces_td_error():
    net = oracle.Net(27, 8, False, (64, 64))
    th = init_params(27, 8, (64, 64), False, seed=41).astype(np.float64)
    e = experiences(1, seed=42)
    out = oracle.dqn_loss_grad(net, th, th, e, 0.99, 1.0, False)
    assert np.array_equal(oracle.sgd(th, out["grad"], 0.0), th)
    w1 = oracle.sgd(th, out["grad"], 1e-3)  # |TD error| decreases for a small alpha
    out1 = oracle.dqn_loss_grad(net, w1, th, e, 0.99, 1.0, False)  # target fixed
    d0 = out["q_s"][0, e["a"][0]] - out["y"][0]
    d1 = out1["q_s"][0, e["a"][0]] - out1["y"][0]
    assert abs(d1) < abs(d0)


def test_ddqn_equals_dqn_right_after_sync():
    # online == target  =>  Q_t(s', argmax_a Q_o(s',a)) = max_a Q_t(s', a)
    net = oracle.Net(27, 8, True, (128,), 512)
    th = init_params(seed=51)
    e = experiences(64, seed=52)
    a = oracle.dqn_loss_grad(net, th, th, e, 0.99, 1.0, False)
    b = oracle.dqn_loss_grad(net, th, th, e, 0.99, 1.0, True)
    assert a["loss"] == b["loss"] and np.array_equal(a["grad"], b["grad"])


def test_learner_target_sync_period():
    # the target net is frozen between syncs and equals the online net right after
    # steps k * period; Q20: sync after the update of step t
    net = oracle.Net(27, 8, False, (64, 64))
    ring = oracle.Ring(1000, 27)
    ring.add(**experiences(500, seed=61))
    ln = oracle.Learner(net, init_params(27, 8, (64, 64), False, seed=62), lr=1e-2,
                        burn_in=100, sync_period=3)
    prev_target = ln.target.copy()
    for t in range(1, 11):
        rc, loss, idx = ln.step(ring, 32)
        assert rc == oracle.OK and np.isfinite(loss)
        if t % 3 == 0:
            assert np.array_equal(ln.target, ln.online)
        else:
            assert np.array_equal(ln.target, prev_target)
            assert not np.array_equal(ln.target, ln.online)
        prev_target = ln.target.copy()
    assert ln.step_count == 10 and ring.events == 10


def test_learner_explicit_sync_target():
    # P:88 / S:306-312: an explicit sync_target() at any step copies the online net bit for bit
    # and the next steps leave the copy frozen (sync_period 0 = manual only); the DDQN
    # bootstrap right after a sync equals the DQN one (online == target makes
    # Q_t(s', argmax Q_o) = max Q_t)
    net = oracle.Net(27, 8, False, (64, 64))
    ring = oracle.Ring(1000, 27)
    ring.add(**experiences(600, seed=63))
    ln = oracle.Learner(net, init_params(27, 8, (64, 64), False, seed=64), lr=1e-2, sync_period=0)
    for _ in range(2):
        assert ln.step(ring, 32)[0] == oracle.OK
    assert not np.array_equal(ln.target, ln.online)
    ln.sync_target()
    assert np.array_equal(ln.target, ln.online)
    frozen = ln.target.copy()
    assert ln.step(ring, 32)[0] == oracle.OK
    assert np.array_equal(ln.target, frozen) and not np.array_equal(ln.online, frozen)
    ln.sync_target()
    rc, b = ring.sample(1, 2, 0, 32)
    assert rc == oracle.OK
    o1 = oracle.dqn_loss_grad(net, ln.online, ln.target, b, 0.99, 1.0, False)
    o2 = oracle.dqn_loss_grad(net, ln.online, ln.target, b, 0.99, 1.0, True)
    assert np.array_equal(o1["y"], o2["y"])


def test_learner_burn_in_leaves_state_untouched():
    net = oracle.Net(27, 8, False, (64, 64))
    ring = oracle.Ring(1000, 27)
    ring.add(**experiences(99, seed=71))
    p0 = init_params(27, 8, (64, 64), False, seed=72)
    ln = oracle.Learner(net, p0, burn_in=100)
    rc, _, _ = ln.step(ring, 32)
    assert rc == oracle.NOT_READY
    assert ring.events == 0 and ln.step_count == 0 and np.array_equal(ln.online, p0)


def test_dyadic_inputs_make_forward_exact_in_fp32():
    # Exact-input mode: dyadic states/weights/rewards and gamma = 0.5 make every
    # forward value, y and delta exactly representable in fp32 -> the GPU must match bitwise
    for net, dy in [(oracle.Net(27, 8, False, (64, 64)), True),
                    (oracle.Net(27, 8, True, (128,), 512), True)]:
        th = init_params(27, 8, net.hidden, net.dueling, net.stream, seed=81, dyadic=True)
        tg = init_params(27, 8, net.hidden, net.dueling, net.stream, seed=82, dyadic=True)
        e = experiences(128, seed=83, dyadic=True)
        for ddqn in (False, True):
            out = oracle.dqn_loss_grad(net, th, tg, e, 0.5, 1.0, ddqn)
            for k in ("q_s", "q_next_target", "y", "z"):
                v = out[k]
                assert np.array_equal(v.astype(np.float32).astype(np.float64), v), k


def test_action_outside_the_action_set_is_rejected():
    # the enumerate-mask select Q[i*A + a_i] is defined only for a_i in [0, A): a batch
    # holding any other action is an argument error, not a silent out-of-bounds read
    net = oracle.Net(state_dim=3, n_actions=4, dueling=True, hidden=(5,), stream=6)
    th = init_params(3, 4, (5,), True, 6, seed=21)
    e = experiences(8, 3, 4, seed=22)
    assert oracle.dqn_loss_grad(net, th, th, e, 0.99, 1.0, False)["loss"] >= 0.0
    for bad in (4, -1):
        e2 = dict(e, a=e["a"].copy())
        e2["a"][5] = bad
        with pytest.raises(ValueError):
            oracle.dqn_loss_grad(net, th, th, e2, 0.99, 1.0, False)
