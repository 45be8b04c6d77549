"""Pins for the oracle's replay ring: layout, FIFO, burn-in, gather/unpack (CPU only).

Checked against the paper's row width, SPEC's worked examples, a brute-force
bounded-deque model and the closed form of FIFO slot ownership.
"""
import collections

import numpy as np
import pytest

import oracle
from inputs import experiences


def _exp(n, D=3, seed=1):
    return experiences(n, state_dim=D, n_actions=8, seed=seed)


def test_row_width_is_paper_57():
    # "the experience replay Variable has shape 1,000,000 by 57" for 27-float states
    r = oracle.Ring(10, 27)
    assert r.rows().shape == (10, 57)


def test_pack_example_spec():
    # D=2, s=[1,2], a=3, r=0.5, s'=[4,5], terminal -> [1,2,4,5,3,0.5,1]
    r = oracle.Ring(4, 2)
    assert r.add([[1, 2]], [3], [0.5], [[4, 5]], [1]) == oracle.OK
    assert r.rows()[0].tolist() == [1, 2, 4, 5, 3, 0.5, 1]
    b = r.gather([0])
    assert b["s"].tolist() == [[1, 2]] and b["s_next"].tolist() == [[4, 5]]
    assert b["a"].tolist() == [3] and b["r"].tolist() == [0.5] and b["done"].tolist() == [1]
    # S:54 zero case
    r0 = oracle.Ring(1, 1)
    r0.add([[0]], [0], [0], [[0]], [0])
    assert r0.rows()[0].tolist() == [0, 0, 0, 0, 0]


def test_unpack_roundtrip_and_corrupt_terminal():
    e = _exp(50, D=5)
    r = oracle.Ring(64, 5)
    assert r.add(**e) == oracle.OK
    b = r.gather(np.arange(50))
    for k in ("s", "a", "r", "s_next", "done"):
        assert np.array_equal(b[k], e[k])  # bit-exact roundtrip
    r.rows()[7, 2 * 5 + 2] = 0.5  # terminal slot 0.5 -> corrupt
    with pytest.raises(ValueError):
        r.gather([7])
    assert r.add(e["s"][:1], e["a"][:1], e["r"][:1], e["s_next"][:1], [2]) == oracle.ECORRUPT


def test_fifo_capacity4_spec_example():
    # capacity 4, add e1..e6 -> holds {e3, e4, e5, e6}
    D = 2
    r = oracle.Ring(4, D)
    for t in range(1, 7):
        assert r.add([[t, t]], [t % 8], [t], [[t, -t]], [0]) == oracle.OK
    held = sorted(r.gather(np.arange(4))["r"].tolist())
    assert held == [3, 4, 5, 6]
    # oldest evicted first: e5 replaced slot 0 (e1), e6 replaced slot 1 (e2)
    assert r.gather([0, 1, 2, 3])["r"].tolist() == [5, 6, 3, 4]
    assert (r.cursor, r.size, r.total) == (2, 4, 6)


def test_k_greater_than_capacity_rejected_without_side_effects():
    r = oracle.Ring(4, 2)
    e = _exp(5, D=2)
    assert r.add(**e) == oracle.EINVAL
    assert (r.cursor, r.size, r.total) == (0, 0, 0)
    e0 = _exp(0, D=2)
    assert r.add(**e0) == oracle.OK  # k = 0 is a no-op
    assert (r.cursor, r.size, r.total) == (0, 0, 0)


def test_fifo_brute_force_random_programs():
    # any add sequence leaves exactly the most recent min(T, C) experiences,
    # compared against a bounded deque; plus the closed form of slot ownership
    #   slot i holds insertion t(i) = i + C * floor((T - 1 - i) / C)   for i < min(T, C).
    g = np.random.default_rng(0)
    for prog in range(2000):
        C = int(g.integers(1, 101))
        r = oracle.Ring(C, 1)
        model = collections.deque(maxlen=C)
        T = 0
        for _ in range(int(g.integers(1, 12))):
            k = int(g.integers(0, C + 1))
            ids = np.arange(T, T + k, dtype=np.float32)
            assert r.add(ids.reshape(-1, 1), np.zeros(k, np.int32), ids, ids.reshape(-1, 1),
                         np.zeros(k, np.uint8)) == oracle.OK
            model.extend(ids.tolist())
            T += k
        n = min(T, C)
        assert r.size == n and r.total == T and r.cursor == T % C
        held = r.gather(np.arange(n))["r"] if n else np.zeros(0)
        assert sorted(held.tolist()) == sorted(model)
        for i in range(n):
            assert held[i] == i + C * ((T - 1 - i) // C)


def test_burn_in_gate_and_c1_schedule():
    # C1: capacity 1000, 7 adds per iteration, burn-in 100 (BASELINE configs[0]).
    # training is skipped during burn-in; nothing advances (Q5).
    D = 27
    r = oracle.Ring(1000, D)
    e = experiences(214 * 7, state_dim=D, seed=1)
    first_ready = None
    wrap_iter = None
    for it in range(1, 215):
        sl = slice((it - 1) * 7, it * 7)
        cur_before = r.cursor
        r.add(e["s"][sl], e["a"][sl], e["r"][sl], e["s_next"][sl], e["done"][sl])
        if r.cursor < cur_before and wrap_iter is None:
            wrap_iter = it
        ev = r.events
        rc, b = r.sample(burn_in=100, seed=2, rank=0, batch=32)
        if r.size < 100:
            assert rc == oracle.NOT_READY and b is None and r.events == ev
        else:
            assert rc == oracle.OK and r.events == ev + 1
            first_ready = first_ready or it
    assert first_ready == 15  # iterations 1-14 hold 7..98 experiences
    assert wrap_iter == 143  # insertions 994..1000 -> slots 994..999, 0
    assert r.events == 214 - 14


def test_sample_matches_sampler_then_gather():
    D = 4
    r = oracle.Ring(300, D)
    e = _exp(450, D=D, seed=7)
    r.add(**{k: v[:300] for k, v in e.items()})
    r.add(**{k: v[300:] for k, v in e.items()})
    rc, b = r.sample(burn_in=1, seed=9, rank=2, batch=33)
    assert rc == oracle.OK
    idx = oracle.sample_indices(9, 2, 0, 300, 33)
    assert np.array_equal(b["idx"], idx)
    # rows by brute force: slot i holds insertion t(i)
    t = np.array([i + 300 * ((450 - 1 - i) // 300) for i in idx])
    assert np.array_equal(b["s"], e["s"][t]) and np.array_equal(b["a"], e["a"][t])
    assert np.array_equal(b["r"], e["r"][t]) and np.array_equal(b["done"], e["done"][t])
    assert np.array_equal(b["s_next"], e["s_next"][t])
    # size 1, batch 4 -> the single experience 4 times
    r1 = oracle.Ring(5, D)
    r1.add(**{k: v[:1] for k, v in e.items()})
    rc, b1 = r1.sample(burn_in=1, seed=1, rank=0, batch=4)
    assert rc == oracle.OK and np.all(b1["idx"] == 0)
    assert np.array_equal(b1["s"], np.repeat(e["s"][:1], 4, axis=0))


# ---- shared-state storage ("by only storing one state per experience, and
# modifying the sample operations"; reading Q30) ----

def test_shared_state_rows_and_next_state():
    # half-width rows [s | a | r | t]; s' of slot i is s of slot i+1; the newest slot has
    # no successor and is never sampled
    D, C = 3, 6
    r = oracle.Ring(C, D, shared=True)
    assert r.rows().shape[1] >= D + 3 and r._r.row_width == D + 3
    e = _exp(4, D)
    assert r.add(e["s"], e["a"], e["r"], None, e["done"]) == oracle.OK
    g = r.gather([0, 1, 2])
    assert np.array_equal(g["s"], e["s"][:3]) and np.array_equal(g["s_next"], e["s"][1:4])
    with pytest.raises(ValueError):
        r.gather([3])   # the newest experience: s' not stored yet


@pytest.mark.parametrize("distinct", [False, True])
def test_shared_state_sampler_brute_force(distinct):
    # the sampler draws logical positions u over the size-1 experiences with a successor,
    # slot = (oldest + u) mod C; checked by brute force against an explicit deque of the
    # stream, before and after the ring wraps
    D, C, B = 2, 40, 16
    r = oracle.Ring(C, D, shared=True, distinct=distinct)
    e = _exp(200, D, seed=3)
    t = 0
    for k in [10, 7, 13, 25, 31, 40, 3]:
        part = {kk: v[t:t + k] for kk, v in e.items()}
        assert r.add(part["s"], part["a"], part["r"], None, part["done"]) == oracle.OK
        t += k
        stream = list(range(max(0, t - C), t))        # experiences in the ring, oldest first
        ev = r.events
        rc, b = r.sample(1, 5, 0, B)
        n = len(stream) - 1
        if distinct and n < B:
            assert rc == oracle.NOT_READY
            continue
        assert rc == oracle.OK
        u = (oracle.sample_distinct if distinct else oracle.sample_indices)(5, 0, ev, n, B)
        for i in range(B):
            src = stream[u[i]]                          # logical position u -> experience
            assert b["idx"][i] == src % C               # its slot (FIFO: t mod C)
            assert np.array_equal(b["s"][i], e["s"][src])
            assert np.array_equal(b["s_next"][i], e["s"][src + 1])   # the next experience's s
            assert b["a"][i] == e["a"][src] and b["done"][i] == e["done"][src]


# ---- P:73 block updates (update-size queue) ---------------------------------------------------
def test_queue_blocks_match_bounded_deque_brute_force():
    # "Experiences are queued in RAM until the queue has enough experiences to update the
    # next block"; brute force: a list queue in front of a bounded deque of written experiences,
    # ragged add sizes (some spanning several blocks) and explicit partial flushes
    import collections
    C, D, U = 12, 5, 4
    ring = oracle.Ring(C, D, update_size=U)
    e = experiences(200, state_dim=D, seed=21)
    queue, written = [], collections.deque(maxlen=C)
    t = 0
    for step, k in enumerate([1, 2, 3, 4, 9, 1, 12, 5, 3, 0, 7, 2, 11]):
        part = {kk: v[t:t + k] for kk, v in e.items()}
        assert ring.add(**part) == oracle.OK
        for j in range(k):
            queue.append(t + j)
            if len(queue) == U:
                written.extend(queue)
                queue = []
        t += k
        if step % 4 == 3:   # explicit partial flush
            n = ring.flush_queue()
            assert n == len(queue)
            written.extend(queue)
            queue = []
        assert ring.queued == len(queue) and ring.size == len(written)
        # ring slots hold the written experiences in FIFO order from the cursor
        g = ring.gather(np.arange(ring.size, dtype=np.int32))
        for i in range(ring.size):
            src = list(written)[(i - ring.cursor) % ring.size] if ring.size == C else list(written)[i]
            assert np.array_equal(g["s"][i], e["s"][src]) and g["a"][i] == e["a"][src]


def test_queue_2000_adds_make_exactly_one_block():
    # P:119 update-size 2,000 with 27-float states: nothing is visible until the 2000th add
    ring = oracle.Ring(10_000, 27, update_size=2000)
    e = experiences(2000, seed=22)
    for i in range(1999):
        assert ring.add(**{k: v[i:i + 1] for k, v in e.items()}) == oracle.OK
    assert ring.size == 0 and ring.queued == 1999 and ring.total == 0
    assert ring.add(**{k: v[1999:] for k, v in e.items()}) == oracle.OK
    assert ring.size == 2000 and ring.queued == 0 and ring.total == 2000 and ring.cursor == 2000


def test_queue_staged_experiences_are_never_sampled():
    # queued experiences are not part of the replay: the sampler draws over the written ones
    ring = oracle.Ring(100, 3, update_size=10)
    e = experiences(25, state_dim=3, seed=23)
    ring.add(**e)   # 2 blocks written, 5 queued
    assert ring.size == 20 and ring.queued == 5
    rc, b = ring.sample(1, 2, 0, 512)
    assert rc == oracle.OK and b["idx"].max() < 20
    staged = {tuple(x) for x in e["s"][20:]}
    assert not any(tuple(x) in staged for x in b["s"])
    rc0 = ring.add(**{k: v[:1] for k, v in e.items()} | {"done": np.array([2], np.uint8)})
    assert rc0 == oracle.ECORRUPT and ring.queued == 5   # nothing queued on a rejected add
