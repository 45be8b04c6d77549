"""Peer-memory data parallelism (dp_peer.cuh, dqn_attach_peers): the gradient mean + SGD in one
kernel that reads every rank's gradient from its memory (P:144 per-step sync).

* `rpl_dp_emulate` runs the kernel for 1 / 2 / 4 / 8 ranks emulated by one cooperative launch on
  this GPU (the publish / wait / read protocol over rank-separate buffers, as the profiling
  recipe prescribes for more ranks than GPUs): every rank's parameters equal the rank-order
  mean-gradient SGD computed here in float32, the ranks stay bit-identical, the two exchange
  slots alternate with the step parity, and a non-finite mean loss skips the update.
* A learner attached to itself (world 1, a real cudaIpc handle) trains bit-identically to an
  unattached one.
"""
import ctypes as C

import numpy as np
import pytest

from inputs import experiences, init_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1801_03138_b200.binding as binding
    return binding


def _slot_stride(P):
    # dp_peer.cuh dp_slot_stride: P + 1 words rounded up to 16 bytes
    return (P + 1 + 3) & ~3


def _xbuf_floats(P):
    flag_off = ((3 * _slot_stride(P) * 4 + 255) // 256) * 256
    return (flag_off + 256) // 4, flag_off // 4


@pytest.mark.parametrize("rs", [0, 1], ids=["all-read", "reduce-scatter"])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_emulated_ranks_mean_sgd(b, world, rs):
    import torch
    P, lr = 5003, np.float32(0.01)
    stride, flag_at = _xbuf_floats(P)
    rng = np.random.default_rng(world)
    xb = torch.zeros(world * stride, dtype=torch.float32, device="cuda")
    w0 = rng.standard_normal(P).astype(np.float32)
    online = torch.from_numpy(np.tile(w0, world)).cuda()
    target = torch.from_numpy(np.tile(w0, world)).cuda()
    gmean = torch.zeros(world * (P + 1), dtype=torch.float32, device="cuda")
    sync = torch.zeros(1, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    w_ref = w0.copy()
    for t in (1, 2, 3):
        slot = (t & 1) * _slot_stride(P)
        grads = rng.standard_normal((world, P + 1)).astype(np.float32)
        for q in range(world):
            xb[q * stride + slot:q * stride + slot + P + 1] = torch.from_numpy(grads[q]).cuda()
        sync.fill_(1 if t == 3 else 0)
        st = b._L.rpl_dp_emulate(world, P, xb.data_ptr(), online.data_ptr(), target.data_ptr(),
                                 gmean.data_ptr(), sync.data_ptr(), err.data_ptr(), C.c_float(lr), t, rs)
        assert st == b.RPL_OK, b.last_error()
        # flags hold the step number
        fl = xb.view(torch.int64)
        for q in range(world):
            assert fl[(q * stride + flag_at) // 2].item() == t
        acc = grads[0].copy()
        for q in range(1, world):
            acc = (acc + grads[q]).astype(np.float32)
        g = (acc / np.float32(world)).astype(np.float32)
        on = online.view(world, P).cpu().numpy()
        gm = gmean.view(world, P + 1).cpu().numpy()
        for q in range(world):   # replicas bit-identical
            assert np.array_equal(on[q], on[0]) and np.array_equal(gm[q], gm[0])
        assert np.array_equal(gm[0], g)   # the mean, in rank order, exactly
        w_ref = (w_ref - lr * g[:P]).astype(np.float32)
        assert np.max(np.abs(on[0] - w_ref)) <= 1e-6 * max(1.0, np.max(np.abs(w_ref)))
        w_ref = on[0].copy()
    tg = target.view(world, P).cpu().numpy()
    assert np.array_equal(tg[0], on[0])   # t = 3 was a sync step
    assert err.item() == 0
    # a non-finite mean loss skips the update and raises the sticky numeric bit
    t = 4
    slot = (t & 1) * _slot_stride(P)
    bad = rng.standard_normal((world, P + 1)).astype(np.float32)
    bad[world - 1, P] = np.nan
    for q in range(world):
        xb[q * stride + slot:q * stride + slot + P + 1] = torch.from_numpy(bad[q]).cuda()
    before = online.clone()
    assert b._L.rpl_dp_emulate(world, P, xb.data_ptr(), online.data_ptr(), target.data_ptr(),
                               gmean.data_ptr(), sync.data_ptr(), err.data_ptr(), C.c_float(lr), t, rs) == b.RPL_OK
    assert torch.equal(online, before) and err.item() == 2


@pytest.mark.parametrize("rs", [0, 1], ids=["all-read", "reduce-scatter"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_ranks_dqn_gradients_vs_oracle_o6(b, world, rs):
    # A10 against the oracle's O6: `world` learners, each with its own
    # replay shard (rank-keyed experience stream and sampler stream), take one Double-DQN step
    # whose per-rank gradient is checked against the oracle (teacher-forced, 1e-5 normwise);
    # the exchange kernel then forms the mean of the GPU gradients and applies SGD on every
    # emulated rank, and the result must equal O6 -- the oracle's rank-order mean of the
    # oracle's per-rank gradients and its SGD -- within 1e-5 normwise per block
    import torch
    import oracle
    from parity import blocks, f32, normwise, step_and_compare
    cfg = b.DQNConfig(max_batch=128, sync_period=0, double_dqn=True, lr=1e-3)
    p0 = init_params(27, 8, (128,), True, 512, seed=3)
    P = p0.size
    stride, _ = _xbuf_floats(P)
    xb = torch.zeros(world * stride, dtype=torch.float32, device="cuda")
    online = torch.from_numpy(np.tile(p0, world)).cuda()
    target = online.clone()
    gmean = torch.zeros(world * (P + 1), dtype=torch.float32, device="cuda")
    sync = torch.zeros(1, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    t = 1
    slot = (t & 1) * _slot_stride(P)
    og, ol = [], []
    for q in range(world):
        rp = b.Replay(3000, 27, seed=2, rank=q)
        orc = oracle.Ring(3000, 27)
        e = experiences(3500, seed=1, rank=q)
        rp.add_many(e)
        orc.add_many(e)
        dqn = b.DQN(cfg, p0)
        out = step_and_compare(b, cfg, dqn, rp, orc, 128, seed=2, rank=q)
        g = np.append(dqn.get_params(b.RPL_GRAD), dqn.debug(b.RPL_DBG_LOSS, 128)[0]).astype(np.float32)
        xb[q * stride + slot:q * stride + slot + P + 1] = torch.from_numpy(g).cuda()
        og.append(out["grad"])
        ol.append(out["loss"])
    assert len({round(float(x), 6) for x in ol}) == world   # distinct shards, distinct batches
    st = b._L.rpl_dp_emulate(world, P, xb.data_ptr(), online.data_ptr(), target.data_ptr(),
                             gmean.data_ptr(), sync.data_ptr(), err.data_ptr(), C.c_float(f32(cfg.lr)), t, rs)
    assert st == b.RPL_OK, b.last_error()
    w_o6, mean_o6 = oracle.dp_mean_sgd(p0, og, f32(cfg.lr))
    on = online.view(world, P).cpu().numpy()
    gm = gmean.view(world, P + 1).cpu().numpy()
    for q in range(world):
        assert np.array_equal(on[q], on[0]) and np.array_equal(gm[q], gm[0])
    for name, sl in blocks(cfg):
        normwise(gm[0][sl], mean_o6[sl], 1e-5, f"mean grad {name}")
        normwise(on[0][sl], w_o6[sl], 1e-5, f"new {name}")
    assert abs(float(gm[0][P]) - float(np.mean(ol))) <= 1e-5 * abs(float(np.mean(ol)))
    assert err.item() == 0


@pytest.mark.parametrize("net,B", [("fast", 128), ("fast", 640), ("generic", 128)])
def test_self_attached_learner_equals_local(b, monkeypatch, net, B):
    # B = 640 takes the tcgen05 step (tc_big.cuh): the peer-memory update rewrites W1 without
    # its bf16 images, so the online images are re-split before the next step and the target's
    # after a sync step
    import torch
    if net == "generic":
        monkeypatch.setenv("RPL_PATH", "generic")
    cfg = b.DQNConfig(max_batch=B, sync_period=4, double_dqn=True, lr=1e-3)
    p0 = init_params(27, 8, (128,), True, 512, seed=3)
    e = experiences(2000, seed=1)
    runs = []
    for attach in (False, True):
        rp = b.Replay(2000, 27, seed=4)
        rp.add_many(e)
        dqn = b.DQN(cfg, p0)
        if attach:
            h = dqn.peer_handle()
            assert len(h) == 64
            dqn.attach_peers(0, 1, h)
        loss = torch.zeros(1, device="cuda")
        for _ in range(7):
            assert dqn.train_step(rp, B, loss) == b.RPL_OK
        torch.cuda.synchronize()
        assert dqn.check() == b.RPL_OK and np.isfinite(loss.item())
        runs.append((dqn.get_params(b.RPL_ONLINE), dqn.get_params(b.RPL_TARGET), loss.item(),
                     dqn.get_params(b.RPL_GRAD)))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])
    assert runs[0][2] == runs[1][2]
    assert np.array_equal(runs[0][3], runs[1][3])


def test_self_attached_wide_learner_equals_local(b):
    # config-5 network (tcgen05 layer 0): the peer-memory update also rewrites W0, whose bf16
    # planes must be re-split before the next forward
    import torch
    D = 84 * 84 * 4
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      max_batch=32, sync_period=3, lr=1e-3)
    from inputs import experiences_u8
    p0 = init_params(D, 8, (128,), True, 512, seed=13)
    e = experiences_u8(64, state_dim=D, seed=12)
    runs = []
    for attach in (False, True):
        rp = b.Replay(64, D, seed=11, state_dtype="u8")
        rp.add(**e)
        dqn = b.DQN(cfg, p0)
        if attach:
            dqn.attach_peers(0, 1, dqn.peer_handle())
        for _ in range(7):   # syncs after steps 3 and 6: the target planes are re-split then only
            assert dqn.train_step(rp, 32) == b.RPL_OK
        assert dqn.check() == b.RPL_OK
        runs.append((dqn.get_params(b.RPL_ONLINE), dqn.get_params(b.RPL_TARGET)))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])


def _ipc_worker(rank, world, port, q):
    # attach only: two processes on one GPU map each other's exchange buffers through cudaIpc
    # (no train step: kernels that wait on one another must not share a GPU)
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1801_03138_b200.binding as b
    from paper_1801_03138_b200 import dp
    dqn = b.DQN(b.DQNConfig(max_batch=32), init_params(27, 8, (128,), True, 512, seed=3))
    try:
        dp.attach_peers(dqn)
        dqn.detach_peers()
        dp.attach_peers(dqn)   # re-attach after a detach
        q.put((rank, "ok"))
    except Exception as ex:   # reported to the parent
        q.put((rank, repr(ex)))
    dqn.detach_peers()
    dist.destroy_process_group()


def test_two_processes_map_each_others_exchange_buffers(b):
    import multiprocessing as mp
    import os
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ps = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
