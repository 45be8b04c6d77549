"""B200-native in-GPU experience replay + fused DQN train step (Parr, arXiv 1801.03138).

The hot path lives in ``lib/libingpu_replay.so`` (hand-written sm_100a CUDA behind the C-ABI
of ``include/ingpu_replay.h``); ``binding`` is its ctypes marshalling layer.
"""
from .binding import (  # noqa: F401
    DQN, DQNConfig, Replay, RplError, dqn_train_step, hidden_units, kernel_launches, last_error,
    nccl_unique_id, replay_add, replay_create, replay_sample, step_flops, sync_target,
)
