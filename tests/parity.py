"""Teacher-forced parity of one GPU train step against the oracle (used by tests/test_gpu_*.py
and __graft_entry__.smoke()).

Per step: the oracle starts from the GPU's fp32 parameters, draws the same Philox batch from
its own ring, and recomputes loss, gradient and the SGD update in fp64.  Sampled indices and
gathered rows must match bit for bit; Q, y, loss, gradients and new weights within `tol`
normwise per tensor (max|gpu - oracle| <= tol * max|oracle|, reading Q24).
Where the GPU took a discrete decision that the oracle would take differently (a ReLU mask
at |z| within rounding of 0, a Double-DQN argmax near-tie) the oracle's own margin must be
within rounding, and the oracle then re-evaluates with the GPU's decision (Q25).
"""
from __future__ import annotations

import numpy as np

import oracle
from inputs import layer_shapes


def f32(x) -> float:
    return float(np.float32(x))


def normwise(g, o, tol, what=""):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    scale = max(float(np.max(np.abs(o))) if o.size else 0.0, 1e-30)
    err = float(np.max(np.abs(g - o))) if o.size else 0.0
    assert err <= tol * scale, f"{what}: max err {err:.3e} > {tol:.1e} * {scale:.3e}"
    return err / scale


def blocks(cfg):
    out, o = [], 0
    for (r, c) in layer_shapes(cfg.state_dim, cfg.n_actions, cfg.hidden, cfg.dueling, cfg.stream):
        out.append((f"W{r}x{c}", slice(o, o + r * c))); o += r * c
        out.append((f"b{r}", slice(o, o + r))); o += r
    return out


def oracle_net(cfg):
    return oracle.Net(cfg.state_dim, cfg.n_actions, cfg.dueling, tuple(cfg.hidden), cfg.stream)


def hidden_layer_slices(cfg):
    sl, o = [], 0
    widths = list(cfg.hidden) + ([2 * cfg.stream] if cfg.dueling else [])
    for w in widths:
        sl.append(slice(o, o + w)); o += w
    return sl


def step_and_compare(b, cfg, dqn, rp, orc_ring, batch, *, seed, rank=0, burn_in=1, tol=1e-5,
                     exact=False, stats=None):
    """One teacher-forced step.  Returns the oracle output dict (or None if NOT_READY)."""
    online = dqn.get_params(b.RPL_ONLINE)
    target = dqn.get_params(b.RPL_TARGET)
    st = dqn.train_step(rp, batch)
    rc, ob = orc_ring.sample(burn_in, seed, rank, batch)
    if rc == oracle.NOT_READY:
        assert st == b.RPL_NOT_READY
        return None
    assert st == b.RPL_OK and rc == oracle.OK
    # bit-exact sample + gather
    for what, key in [(b.RPL_DBG_IDX, "idx"), (b.RPL_DBG_S, "s"), (b.RPL_DBG_S_NEXT, "s_next"),
                      (b.RPL_DBG_A, "a"), (b.RPL_DBG_R, "r"), (b.RPL_DBG_DONE, "done")]:
        g = dqn.debug(what, batch)
        assert np.array_equal(g.view(np.uint8), np.ascontiguousarray(ob[key]).view(np.uint8)), key
    net = oracle_net(cfg)
    gamma, kappa = f32(cfg.gamma), (np.inf if np.isinf(cfg.huber_kappa) else f32(cfg.huber_kappa))
    if ob["s"].dtype == np.uint8:   # byte states: the network input is u8 / 255 (Q27)
        ob = dict(ob, s=oracle.u8_input(ob["s"]), s_next=oracle.u8_input(ob["s_next"]))
    out = oracle.dqn_loss_grad(net, online, target, ob, gamma, kappa, cfg.double_dqn)
    # decision replay (Q25)
    H = net.hidden_units
    hg = dqn.debug(b.RPL_DBG_H, batch, H)
    mask_g = (hg > 0).astype(np.uint8)
    flips = mask_g != out["on"]
    override = False
    if flips.any():
        for sl in hidden_layer_slices(cfg):
            z = out["z"][:, sl]
            f = flips[:, sl]
            if f.any():
                scale = np.max(np.abs(z), axis=1, keepdims=True)
                bad = f & (np.abs(z) > max(tol, 1e-5) * scale)
                assert not bad.any(), f"ReLU decision differs beyond rounding: z={z[bad][:4]}"
        override = True
    astar = None
    if cfg.double_dqn:
        ag = dqn.debug(b.RPL_DBG_ASTAR, batch)
        if not np.array_equal(ag, out["a_star"]):
            qo = out["q_next_online"]
            rows = np.nonzero(ag != out["a_star"])[0]
            for i in rows:
                margin = qo[i, out["a_star"][i]] - qo[i, ag[i]]
                assert margin <= max(tol, 1e-5) * max(1.0, np.max(np.abs(qo[i]))), "argmax beyond rounding"
            astar = ag
            override = True
    if override:
        out = oracle.dqn_loss_grad(net, online, target, ob, gamma, kappa, cfg.double_dqn,
                                   mask_override=mask_g, argmax_override=astar)
    if stats is not None:
        stats["mask_flips"] = stats.get("mask_flips", 0) + int(flips.sum())
        stats["steps"] = stats.get("steps", 0) + 1
    loss_g = dqn.debug(b.RPL_DBG_LOSS, batch)[0]
    qg = dqn.debug(b.RPL_DBG_Q, batch)
    qtg = dqn.debug(b.RPL_DBG_QT_NEXT, batch)
    yg = dqn.debug(b.RPL_DBG_Y, batch)
    grad_g = dqn.get_params(b.RPL_GRAD)
    new_g = dqn.get_params(b.RPL_ONLINE)
    new_o = oracle.sgd(online, out["grad"], f32(cfg.lr))
    if exact:
        assert np.array_equal(qg.astype(np.float64), out["q_s"])
        assert np.array_equal(qtg.astype(np.float64), out["q_next_target"])
        assert np.array_equal(yg.astype(np.float64), out["y"])
        if cfg.double_dqn:
            assert np.array_equal(dqn.debug(b.RPL_DBG_QO_NEXT, batch).astype(np.float64),
                                  out["q_next_online"])
            assert np.array_equal(dqn.debug(b.RPL_DBG_ASTAR, batch), out["a_star"])
        assert np.array_equal(hg.astype(np.float64), out["z"] * out["on"])
    normwise(qg, out["q_s"], tol, "Q(s)")
    normwise(qtg, out["q_next_target"], tol, "Q_target(s')")
    if cfg.double_dqn:
        normwise(dqn.debug(b.RPL_DBG_QO_NEXT, batch), out["q_next_online"], tol, "Q_online(s')")
    normwise(yg, out["y"], tol, "y")
    assert abs(float(loss_g) - out["loss"]) <= tol * max(abs(out["loss"]), 1e-30), "loss"
    for name, sl in blocks(cfg):
        if np.max(np.abs(out["grad"][sl])) > 0:
            normwise(grad_g[sl], out["grad"][sl], tol, f"grad {name}")
        normwise(new_g[sl], new_o[sl], tol, f"new {name}")
    out["online_before"] = online
    out["target_before"] = target
    return out
