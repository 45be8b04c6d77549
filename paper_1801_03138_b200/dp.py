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


def shard_seed(base: int, rank: int) -> tuple[int, int]:
    """(data seed, sampler rank) of a learner: every rank draws its own experience stream and
    its own Philox sampler stream (the rank goes into counter word 3, Q3)."""
    return base, rank
