"""World-size-2 CPU (gloo) tests of the data-parallel host logic.

The GPU path all-reduces the flat gradient with NCCL inside dqn_train_step; here the same
protocol runs with the oracle as the per-rank learner and gloo as the transport:
  * the 128-byte NCCL-id broadcast used by paper_1801_03138_b200.dp reaches every rank intact;
  * replicas stay bit-identical step after step (mean of per-rank gradients, same SGD);
  * world 2 with identical shards and a rank-independent stream equals one learner bit for
    bit ((g + g) / 2 == g exactly);
  * with distinct shards the averaged update equals the rank-order mean (O6 reading Q23).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from inputs import experiences, init_params

NET = oracle.Net(27, 8, False, (64, 64))
STEPS = 5
B = 32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _learner_steps(rank, world, same_shard, out):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1801_03138_b200 import dp
    # 1. unique-id broadcast
    payload = bytes(range(128)) if rank == 0 else None
    got = dp.broadcast_bytes(payload, 0)
    assert got == bytes(range(128))
    # 2. per-rank shard + sampler stream
    data_rank = 0 if same_shard else rank
    ring = oracle.Ring(500, 27)
    ring.add(**experiences(500, seed=1, rank=data_rank))
    w = init_params(27, 8, (64, 64), False, seed=3).astype(np.float64)
    tg = w.copy()
    for step in range(STEPS):
        rc, batch = ring.sample(1, 2, data_rank, B)
        assert rc == oracle.OK
        o = oracle.dqn_loss_grad(NET, w.astype(np.float32), tg.astype(np.float32), batch, 0.99, 1.0, False)
        g = torch.from_numpy(o["grad"].copy())
        dist.all_reduce(g, op=dist.ReduceOp.SUM)
        g = g.numpy() / world
        w = oracle.sgd(w, g, 1e-2).astype(np.float32).astype(np.float64)
        gathered = [torch.zeros_like(torch.from_numpy(w)) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(w))
        assert all(np.array_equal(x.numpy(), w) for x in gathered), "replicas diverged"
    out[rank] = w
    dist.destroy_process_group()


def _run(world, same_shard):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_learner_steps, args=(world, same_shard, out), nprocs=world, join=True)
        return {k: v for k, v in out.items()}


def _single(data_rank):
    ring = oracle.Ring(500, 27)
    ring.add(**experiences(500, seed=1, rank=data_rank))
    w = init_params(27, 8, (64, 64), False, seed=3).astype(np.float64)
    tg = w.copy()
    grads = []
    for step in range(STEPS):
        rc, batch = ring.sample(1, 2, data_rank, B)
        o = oracle.dqn_loss_grad(NET, w.astype(np.float32), tg.astype(np.float32), batch, 0.99, 1.0, False)
        w = oracle.sgd(w, o["grad"], 1e-2).astype(np.float32).astype(np.float64)
        grads.append(o["grad"])
    return w


def test_world2_identical_shards_equals_single_learner():
    out = _run(2, same_shard=True)
    assert np.array_equal(out[0], out[1])
    assert np.array_equal(out[0], _single(0))


def test_world2_distinct_shards_replicas_identical_and_mean_rule():
    out = _run(2, same_shard=False)
    assert np.array_equal(out[0], out[1])
    # the first averaged step equals the rank-order mean of the two per-rank gradients
    w0 = init_params(27, 8, (64, 64), False, seed=3)
    gs = []
    for r in (0, 1):
        ring = oracle.Ring(500, 27)
        ring.add(**experiences(500, seed=1, rank=r))
        rc, batch = ring.sample(1, 2, r, B)
        gs.append(oracle.dqn_loss_grad(NET, w0, w0, batch, 0.99, 1.0, False)["grad"])
    assert not np.array_equal(gs[0], gs[1])      # the shards really differ
    assert not np.array_equal(out[0], _single(0))


# ---- periodic parameter averaging ("each GPU could have its own model that is
# synchronized periodically ... iterative parameter mixing"; avg_period, reading Q31) ----
AVG_K = 2


def _mixing_steps(rank, world, out):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ring = oracle.Ring(500, 27)
    ring.add(**experiences(500, seed=1, rank=rank))
    w = init_params(27, 8, (64, 64), False, seed=3).astype(np.float32)
    tg = w.copy()
    hist, same = [], []
    for step in range(1, STEPS + 1):
        rc, batch = ring.sample(1, 2, rank, B)
        o = oracle.dqn_loss_grad(NET, w, tg, batch, 0.99, 1.0, False)
        w = oracle.sgd(w, o["grad"], 1e-2).astype(np.float32)          # local SGD
        if step % AVG_K == 0:                                           # mean over ranks
            for arr in (w, tg):
                t = torch.from_numpy(arr)
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
                arr[...] = (t / world).numpy()
        gathered = [torch.zeros_like(torch.from_numpy(w)) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(w))
        same.append(all(np.array_equal(x.numpy(), w) for x in gathered))
        hist.append(w.copy())
    out[rank] = (hist, same)
    dist.destroy_process_group()


def test_world2_periodic_parameter_averaging():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_mixing_steps, args=(2, out), nprocs=2, join=True)
        res = {k: v for k, v in out.items()}
    # replicas agree exactly right after every mixing step and differ in between
    for step, same in enumerate(res[0][1], start=1):
        assert same == (step % AVG_K == 0), step
    # the first mixed weights are the mean of the two ranks' local trajectories
    local = []
    for r in (0, 1):
        ring = oracle.Ring(500, 27)
        ring.add(**experiences(500, seed=1, rank=r))
        w = init_params(27, 8, (64, 64), False, seed=3).astype(np.float32)
        tg = w.copy()
        for _ in range(AVG_K):
            rc, batch = ring.sample(1, 2, r, B)
            w = oracle.sgd(w, oracle.dqn_loss_grad(NET, w, tg, batch, 0.99, 1.0, False)["grad"],
                           1e-2).astype(np.float32)
        local.append(w)
    assert not np.array_equal(local[0], local[1])
    np.testing.assert_array_equal(res[0][0][AVG_K - 1], (local[0] + local[1]) / np.float32(2))


def _gather_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1801_03138_b200 import dp
    payload = bytes([rank * 16 + i % 16 for i in range(64)])
    q.put((rank, dp.gather_bytes(payload, 64)))
    dist.destroy_process_group()


def test_world2_peer_handle_allgather():
    # dqn_attach_peers' handle exchange: every rank receives all ranks' 64-byte handles,
    # concatenated in rank order
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    want = bytes([i % 16 for i in range(64)]) + bytes([16 + i % 16 for i in range(64)])
    assert out[0] == want and out[1] == want


class _MockLearner:
    def __init__(self, rank, fail):
        self.rank, self.fail, self.calls = rank, fail, []

    def peer_handle(self):
        return bytes([self.rank]) * 64

    def attach_peers(self, rank, world, handles):
        self.calls.append(("attach_peers", handles))
        if self.fail:
            raise RuntimeError("IPC mapping failed")

    def detach_peers(self):
        self.calls.append(("detach_peers",))


def _auto_worker(rank, world, port, fail_rank, peer_ok, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1801_03138_b200 import dp
    m = _MockLearner(rank, rank == fail_rank)
    dp.attach = lambda dqn: dqn.calls.append(("nccl",))   # no NCCL on this CPU box
    q.put((rank, dp.attach_auto(m, peer_ok=peer_ok), [c[0] for c in m.calls]))
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank,peer_ok,want", [(-1, True, "p2p"), (1, True, "nccl"), (-1, False, "nccl")])
def test_world2_attach_auto_agrees(fail_rank, peer_ok, want):
    # every rank takes the same data-parallel path: peer memory only when all ranks can map all
    # peers; one failed mapping sends everyone (the mapped ranks detaching first) to NCCL
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_auto_worker, args=(r, 2, port, fail_rank, peer_ok, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, path, calls = q.get(timeout=120)
        res[r] = (path, calls)
    for p in ps:
        p.join(timeout=60)
    assert res[0][0] == res[1][0] == want
    if want == "p2p":
        assert res[0][1] == res[1][1] == ["attach_peers"]
    elif peer_ok:
        assert res[0][1] == ["attach_peers", "detach_peers", "nccl"] and res[1][1] == ["attach_peers", "nccl"]
    else:
        assert res[0][1] == res[1][1] == ["nccl"]
