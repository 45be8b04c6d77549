"""B200-native in-GPU experience replay + fused DQN train step (Parr, arXiv 1801.03138).

The hot path lives in ``lib/libingpu_replay.so`` (hand-written sm_100a CUDA behind the C-ABI
of ``include/ingpu_replay.h``); ``binding`` is its ctypes marshalling layer.  The package
imports without the library (so ``paper_1801_03138_b200.build`` can create it); the first use
of a binding name loads it and raises ImportError if it is missing -- there is no CPU fallback.
"""
_EXPORTS = (
    "DQN", "DQNConfig", "Replay", "RplError", "dqn_train_step", "hidden_units", "kernel_launches",
    "last_error", "nccl_unique_id", "replay_add", "replay_create", "replay_sample", "step_flops",
    "sync_target",
)


def __getattr__(name):
    if name in _EXPORTS:
        from . import binding
        return getattr(binding, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
