"""Seeded synthetic Melee-shaped experiences and parameter blobs.

Recipe (the paper's Melee data is not available):
  * states s, s' : `state_dim` float32 values U[-1, 1)   (27 normalised game-memory
    floats per state, P:71 [Methods]),
  * action a     : uniform integer in [0, n_actions)     (controller presses),
  * reward r     : float32 U[-1, 1),
  * terminal     : Bernoulli(1/64) as uint8 {0, 1}.
Parameters: Glorot-uniform weights +-sqrt(6/(fan_in+fan_out)) per layer, biases
U(-0.05, 0.05) (the paper gives no initialisation; SPEC S:335 uses Glorot).

"Dyadic" variants draw every value from a small set of dyadic rationals so that all fp32
forward arithmetic is exact.

Every stream is numpy's Philox bit generator keyed by (seed, rank, purpose); nothing here
is shared arithmetic of the method.
"""
from __future__ import annotations

import numpy as np

PURPOSE_DATA = 1
PURPOSE_INIT = 2
PURPOSE_AUX = 3


def rng(seed: int, rank: int = 0, purpose: int = PURPOSE_DATA) -> np.random.Generator:
    key = (int(seed) & 0xFFFFFFFF) | ((int(rank) & 0xFFFFFF) << 32) | (int(purpose) << 56)
    return np.random.Generator(np.random.Philox(key=key))


def experiences(n: int, state_dim: int = 27, n_actions: int = 8, seed: int = 1, rank: int = 0,
                done_prob: float = 1.0 / 64.0, dyadic: bool = False) -> dict:
    """n synthetic experiences as SoA numpy arrays (s, a, r, s_next, done)."""
    g = rng(seed, rank, PURPOSE_DATA)
    if dyadic:
        # multiples of 1/4 in [-1, 1) and rewards in multiples of 1/8 in [-1, 1)
        s = (g.integers(-4, 4, size=(n, state_dim)) / 4.0).astype(np.float32)
        s2 = (g.integers(-4, 4, size=(n, state_dim)) / 4.0).astype(np.float32)
        r = (g.integers(-8, 8, size=n) / 8.0).astype(np.float32)
    else:
        s = g.uniform(-1.0, 1.0, size=(n, state_dim)).astype(np.float32)
        s2 = g.uniform(-1.0, 1.0, size=(n, state_dim)).astype(np.float32)
        r = g.uniform(-1.0, 1.0, size=n).astype(np.float32)
    a = g.integers(0, n_actions, size=n).astype(np.int32)
    done = (g.random(n) < done_prob).astype(np.uint8)
    return dict(s=s, a=a, r=r, s_next=s2, done=done)


ATARI_STATE_DIM = 84 * 84 * 4   # SURVEY config 5: 84x84x4 uint8 frames stacked per state


# ---- counter-based byte rows: experience t is a pure function of t (large rings) -----------
# Rings too large to generate and keep on the host (configs[4]: 56 GB at 1M rows) are filled
# from this hash on the device (torch) and checked on the host (numpy) for the sampled rows
# only; both evaluate the same 32-bit integer arithmetic.
_M = 0xFFFFFFFF


def _h32(x, xp):
    x = x & _M
    x = (x ^ (x >> 16)) & _M
    x = (x * 0x7FEB352D) & _M
    x = (x ^ (x >> 15)) & _M
    x = (x * 0x846CA68B) & _M
    return (x ^ (x >> 16)) & _M


def _u8_fields(t, D, n_actions, xp, arange):
    j = arange(D)[None, :]
    tt = t[:, None]
    s = _h32(tt * 0x9E3779B1 + j * 0x85EBCA77 + 0x1000, xp) & 0xFF
    s2 = _h32(tt * 0x9E3779B1 + j * 0x85EBCA77 + 0x2000, xp) & 0xFF
    ha = _h32(t * 0x9E3779B1 + 0x3000, xp)
    hr = _h32(t * 0x9E3779B1 + 0x4000, xp)
    hd = _h32(t * 0x9E3779B1 + 0x5000, xp)
    return s, s2, ha % n_actions, hr >> 8, (hd < (1 << 26))


def u8_rows_np(t, state_dim: int = ATARI_STATE_DIM, n_actions: int = 8) -> dict:
    """Experiences number t (int array) of the counter-based byte stream, as numpy arrays."""
    t = np.asarray(t, dtype=np.int64)
    s, s2, a, r24, d = _u8_fields(t, state_dim, n_actions, np, lambda n: np.arange(n, dtype=np.int64))
    r = (r24.astype(np.float64) * 2.0 ** -23 - 1.0).astype(np.float32)
    return dict(s=s.astype(np.uint8), a=a.astype(np.int32), r=r, s_next=s2.astype(np.uint8),
                done=d.astype(np.uint8))


def u8_rows_torch(t, state_dim: int = ATARI_STATE_DIM, n_actions: int = 8) -> dict:
    """The same experiences as CUDA tensors (t: int64 tensor on the device)."""
    import torch
    s, s2, a, r24, d = _u8_fields(t, state_dim, n_actions, torch,
                                  lambda n: torch.arange(n, dtype=torch.int64, device=t.device))
    r = (r24.to(torch.float64) * 2.0 ** -23 - 1.0).to(torch.float32)
    return dict(s=s.to(torch.uint8), a=a.to(torch.int32), r=r, s_next=s2.to(torch.uint8),
                done=d.to(torch.uint8))


def experiences_u8(n: int, state_dim: int = ATARI_STATE_DIM, n_actions: int = 8, seed: int = 1,
                   rank: int = 0, done_prob: float = 1.0 / 64.0) -> dict:
    """n synthetic Atari-shaped experiences (SURVEY config 5): uint8 states uniform over
    [0, 255], actions / rewards / terminals as in `experiences`."""
    g = rng(seed, rank, PURPOSE_DATA)
    s = g.integers(0, 256, size=(n, state_dim), dtype=np.uint8)
    s2 = g.integers(0, 256, size=(n, state_dim), dtype=np.uint8)
    r = g.uniform(-1.0, 1.0, size=n).astype(np.float32)
    a = g.integers(0, n_actions, size=n).astype(np.int32)
    done = (g.random(n) < done_prob).astype(np.uint8)
    return dict(s=s, a=a, r=r, s_next=s2, done=done)


def layer_shapes(state_dim: int, n_actions: int, hidden, dueling: bool, stream: int = 512):
    """(out, in) of every weight matrix of the parameter blob, in blob order
    (DESIGN.md "Parameter blob"); each W [out x in] is followed by its bias [out]."""
    shapes = []
    k = state_dim
    for h in hidden:
        shapes.append((h, k))
        k = h
    if dueling:
        shapes.append((2 * stream, k))        # [V stream ; A stream] hidden layers
        shapes.append((1 + n_actions, stream))  # [V head ; A head]
    else:
        shapes.append((n_actions, k))
    return shapes


def init_params(state_dim: int = 27, n_actions: int = 8, hidden=(128,), dueling: bool = True,
                stream: int = 512, seed: int = 3, dyadic: bool = False,
                bias_scale: float = 0.05) -> np.ndarray:
    """A flat float32 parameter blob (Glorot-uniform weights, small uniform biases)."""
    g = rng(seed, 0, PURPOSE_INIT)
    parts = []
    for li, (o, i) in enumerate(layer_shapes(state_dim, n_actions, hidden, dueling, stream)):
        if dyadic:
            den = 16.0 if dueling else 8.0
            W = g.integers(-1, 2, size=(o, i)) / den
            b = g.integers(-1, 2, size=o) / den
        else:
            fan_in, fan_out = i, o
            if dueling and li == len(hidden):       # each stream is its own layer
                fan_out = stream
            if dueling and li == len(hidden) + 1:   # V head (1) / A head (A)
                fan_out = n_actions
            lim = np.sqrt(6.0 / (fan_in + fan_out))
            W = g.uniform(-lim, lim, size=(o, i))
            b = g.uniform(-bias_scale, bias_scale, size=o)
        parts.append(W.astype(np.float32).ravel())
        parts.append(b.astype(np.float32).ravel())
    return np.concatenate(parts)
