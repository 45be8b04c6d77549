"""Data-parallel learners ("the agent's model would have to be synchronized every train
step"): one process per GPU, each with its own replay shard and sampler stream (rank in the
Philox counter), one gradient all-reduce (mean, NCCL over NVLink/NVSwitch) per step inside
``dqn_train_step`` once the learner is attached.

Host-side plumbing only: the NCCL communicator is created by the C library from a 128-byte
unique id that rank 0 generates and ``torch.distributed`` broadcasts.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def broadcast_bytes(payload: bytes | None, src: int = 0, nbytes: int = 128) -> bytes:
    """Broadcast `nbytes` from `src` over the default process group (gloo: CPU tensor,
    nccl: CUDA tensor)."""
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    if dist.get_rank() == src:
        assert payload is not None and len(payload) == nbytes
        buf.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(buf, src)
    return bytes(buf.cpu().numpy().tobytes())


def attach(dqn) -> None:
    """Attach a learner (binding.DQN) to an NCCL communicator spanning the default group."""
    from . import binding
    rank, world = dist.get_rank(), dist.get_world_size()
    if world == 1:
        return
    uid = binding.nccl_unique_id() if rank == 0 else None
    dqn.attach_nccl(rank, world, broadcast_bytes(uid, 0))


def gather_bytes(payload: bytes, nbytes: int = 64) -> bytes:
    """All-gather `nbytes` from every rank over the default process group; the result is the
    ranks' payloads concatenated in rank order."""
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    assert len(payload) == nbytes
    mine = torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(dev)
    out = [torch.zeros(nbytes, dtype=torch.uint8, device=dev) for _ in range(dist.get_world_size())]
    dist.all_gather(out, mine)
    return b"".join(bytes(t.cpu().numpy().tobytes()) for t in out)


def attach_peers(dqn) -> None:
    """Attach a learner to its node's peers through peer memory (dqn_attach_peers): the
    gradient mean and SGD then run in one kernel reading every rank's gradient over NVLink."""
    rank, world = dist.get_rank(), dist.get_world_size()
    dqn.attach_peers(rank, world, gather_bytes(dqn.peer_handle(), 64))


def attach_auto(dqn, peer_ok: bool | None = None) -> str:
    """Peer memory when every rank can map every other rank's buffer (one node, peer access
    between all the ranks' GPUs), else NCCL; every rank takes the same choice.  Returns
    "p2p" or "nccl".  (peer_ok overrides the peer-access probe; tests.)"""
    rank, world = dist.get_rank(), dist.get_world_size()
    if world == 1:
        return "none"
    ok = world <= 8 if peer_ok is None else peer_ok
    if ok and peer_ok is None:
        dev = torch.cuda.current_device()
        n = torch.cuda.device_count()
        ok = n >= world and all(torch.cuda.can_device_access_peer(dev, o) for o in range(world) if o != dev)
    # every rank runs the same collectives whatever fails locally: agree on the probe, then on
    # the exported handles, then on the mappings
    if not _all_min(1 if ok else 0):
        attach(dqn)
        return "nccl"
    handle, h_ok = bytes(64), True
    try:
        handle = dqn.peer_handle()
    except Exception:
        h_ok = False
    if not _all_min(1 if h_ok else 0):
        attach(dqn)
        return "nccl"
    handles = gather_bytes(handle, 64)
    attached = True
    try:
        dqn.attach_peers(rank, world, handles)
    except Exception:
        attached = False
    if _all_min(1 if attached else 0):
        return "p2p"
    if attached:
        dqn.detach_peers()
    attach(dqn)
    return "nccl"


def _all_min(v: int) -> int:
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([v], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return int(t.item())


def shard_seed(base: int, rank: int) -> tuple[int, int]:
    """(data seed, sampler rank) of a learner: every rank draws its own experience stream and
    its own Philox sampler stream (the rank goes into counter word 3, Q3)."""
    return base, rank
