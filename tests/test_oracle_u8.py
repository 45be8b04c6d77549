"""Pins for the oracle's byte-state replay and network input (SURVEY config 5; CPU only).

The u8 ring must be the float ring's FIFO / sampler / gather over byte states,
checked against a brute-force bounded deque; the input map x = u8 / 255 (reading Q27) is
pinned by its exact values and by the exactly rounded fp32 quotient.
"""
import collections
from fractions import Fraction

import numpy as np

import oracle
from inputs import experiences_u8


def test_u8_ring_fifo_matches_bounded_deque():
    # P:73 "the oldest experiences are overwritten": brute force with a bounded deque of
    # (slot-order) experiences over ragged add sizes that wrap the ring several times
    C, D = 7, 33
    ring = oracle.RingU8(C, D)
    e = experiences_u8(60, state_dim=D, seed=5)
    slots = [None] * C
    cursor, size, t = 0, 0, 0
    for k in [1, 3, 7, 2, 5, 6, 1, 4, 7, 7, 3, 2, 5, 7]:
        part = {key: v[t:t + k] for key, v in e.items()}
        assert ring.add(**part) == oracle.OK
        for j in range(k):
            slots[cursor] = t + j
            cursor = (cursor + 1) % C
            size = min(size + 1, C)
        t += k
        assert (ring.cursor, ring.size, ring.total) == (cursor, size, t)
        idx = np.arange(size, dtype=np.int32)
        g = ring.gather(idx)
        for i in range(size):
            src = slots[i]
            assert np.array_equal(g["s"][i], e["s"][src])
            assert np.array_equal(g["s_next"][i], e["s_next"][src])
            assert g["a"][i] == e["a"][src] and g["r"][i] == e["r"][src]
            assert g["done"][i] == e["done"][src]
    assert ring.add(**{key: v[:C + 1] for key, v in e.items()}) == oracle.EINVAL   # k > C


def test_u8_ring_sampler_is_the_float_rings_sampler():
    # the same Philox stream (Q3) and burn-in gate as the float ring
    C, D = 50, 16
    ring = oracle.RingU8(C, D)
    e = experiences_u8(30, state_dim=D, seed=6)
    ring.add(**{k: v[:10] for k, v in e.items()})
    rc, _ = ring.sample(20, 2, 3, 8)
    assert rc == oracle.NOT_READY and ring.events == 0
    ring.add(**{k: v[10:] for k, v in e.items()})
    for ev in range(3):
        rc, b = ring.sample(20, 2, 3, 64)
        assert rc == oracle.OK
        assert np.array_equal(b["idx"], oracle.sample_indices(2, 3, ev, 30, 64))
        assert np.array_equal(b["s"], e["s"][b["idx"]])
        assert np.array_equal(b["s_next"], e["s_next"][b["idx"]])


def test_u8_input_is_the_rounded_quotient():
    # Q27: x = u8 / 255 -> the fp32 nearest the exact rational u/255 for every byte value
    u = np.arange(256, dtype=np.uint8)
    x = oracle.u8_input(u)
    assert x[0] == 0.0 and x[255] == 1.0 and x[51] == np.float32(0.2)
    for v in range(256):
        q = Fraction(v, 255)
        f = Fraction(float(x[v]))
        # no fp32 neighbour is closer to the exact quotient
        up = Fraction(float(np.nextafter(x[v], np.float32(2))))
        dn = Fraction(float(np.nextafter(x[v], np.float32(-1))))
        assert abs(f - q) <= abs(up - q) and abs(f - q) <= abs(dn - q)
    assert np.all(np.diff(x) > 0)
