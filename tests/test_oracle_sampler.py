"""Pins for the oracle's Philox generator and index sampler (CPU only).

Each check is against something other than the oracle itself: published known-answer
vectors, the paper's duplicate rate, closed-form probabilities and chi-square
statistics.
"""
import math
import os

import numpy as np
import pytest
from scipy import stats

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _kat())
def test_philox_known_answer(ctr, key, expect):
    # Random123 examples/kat_vectors (golden/philox4x32_10_kat.txt)
    out = oracle.philox4x32_10(ctr, key)
    assert [int(x) for x in out] == expect


@pytest.mark.parametrize("n", [1, 2, 3, 7, 10, 1000, 999_983, 1_000_000, 2**31 - 1])
def test_indices_in_range(n):
    # P:75 "integers uniformly between 0 and the current size": half-open [0, n) (Q1)
    for event in (0, 1, 2**32 + 5):
        idx = oracle.sample_indices(seed=2, rank=0, event=event, n=n, batch=4099)
        assert idx.min() >= 0 and idx.max() < n
    if n == 1:
        assert np.all(idx == 0)  # the single experience every time


def test_events_and_ranks_give_distinct_streams():
    a = oracle.sample_indices(2, 0, 0, 1_000_000, 256)
    b = oracle.sample_indices(2, 0, 1, 1_000_000, 256)
    c = oracle.sample_indices(2, 1, 0, 1_000_000, 256)
    d = oracle.sample_indices(3, 0, 0, 1_000_000, 256)
    for x in (b, c, d):
        assert np.mean(a == x) < 0.01
    # deterministic: same (seed, rank, event) -> same batch
    assert np.array_equal(a, oracle.sample_indices(2, 0, 0, 1_000_000, 256))
    # a batch is a prefix-stable function of i (index i depends only on Philox call i/2)
    assert np.array_equal(oracle.sample_indices(2, 0, 0, 1_000_000, 7), a[:7])


def test_uniform_chi_square():
    # per-index frequencies over [0, 10) uniform within the chi-square 99% bound
    n, draws = 10, 100_000
    idx = oracle.sample_indices(seed=2, rank=0, event=11, n=n, batch=draws)
    counts = np.bincount(idx, minlength=n)
    chi2 = ((counts - draws / n) ** 2 / (draws / n)).sum()
    assert chi2 < stats.chi2.ppf(0.99, df=n - 1)
    # also non-power-of-two n with a large range: equal-width bins
    n2 = 999_983
    idx2 = oracle.sample_indices(seed=5, rank=3, event=0, n=n2, batch=200_000)
    bins = np.bincount((idx2.astype(np.int64) * 20) // n2, minlength=20)
    chi2b = ((bins - 10_000) ** 2 / 10_000).sum()
    assert chi2b < stats.chi2.ppf(0.99, df=19)


def test_duplicate_rate_matches_paper():
    # P:75 [Methods]: with replacement, a batch of 32 from 1,000,000 contains a duplicate
    # "0.05% of the time".  Birthday product 1 - prod_{i<32} (1 - i/1e6) = 4.9588e-4.
    analytic = 1.0 - math.prod(1.0 - i / 1e6 for i in range(32))
    assert abs(analytic - 4.9588e-4) < 1e-7
    assert round(analytic * 100, 2) == 0.05
    # Monte Carlo over 10^6 batches of 32: within [3.5e-4, 6.5e-4]
    groups = 1_000_000
    idx = oracle.sample_indices(seed=2, rank=0, event=0, n=1_000_000, batch=32 * groups)
    g = np.sort(idx.reshape(groups, 32), axis=1)
    dup = np.any(g[:, 1:] == g[:, :-1], axis=1).mean()
    assert 3.5e-4 <= dup <= 6.5e-4
    # and per-event batches (the way the train step draws them) over 20,000 events at n=1000
    # (C1's ring): P(dup) = 1 - prod_{i<32}(1 - i/1000) = 0.3914
    n_ev = 20_000
    d = 0
    for e in range(n_ev):
        b = np.sort(oracle.sample_indices(2, 0, e, 1000, 32))
        d += bool(np.any(b[1:] == b[:-1]))
    p = 1.0 - math.prod(1.0 - i / 1000 for i in range(32))
    se = math.sqrt(p * (1 - p) / n_ev)
    assert abs(d / n_ev - p) < 4 * se


# ---- distinct sampling ("I plan on switching back to sampling distinct integers";
# SURVEY 8(f) NEXT-4; reading Q29: the first B distinct values of the same index stream) ----

def _stream(seed, rank, event, n, length):
    # the uniform sampler's stream extended past B: position t is index t of a batch of `length`
    return oracle.sample_indices(seed, rank, event, n, length)


@pytest.mark.parametrize("n,B", [(1_000_000, 128), (200, 128), (128, 128), (37, 5), (1000, 999)])
def test_distinct_is_first_distinct_of_stream(n, B):
    idx = oracle.sample_distinct(2, 3, 7, n, B)
    assert len(set(idx.tolist())) == B and idx.min() >= 0 and idx.max() < n
    # brute force over a long enough prefix of the uniform stream
    L = 64
    while True:
        st = _stream(2, 3, 7, n, L)
        firsts = list(dict.fromkeys(st.tolist()))
        if len(firsts) >= B:
            break
        L *= 2
    assert idx.tolist() == firsts[:B]


def test_distinct_equals_uniform_without_collisions():
    # with no repeated index in the uniform batch the two samplers agree exactly
    for ev in range(20):
        u = oracle.sample_indices(2, 0, ev, 1_000_000, 64)
        if len(set(u.tolist())) == 64:
            assert np.array_equal(oracle.sample_distinct(2, 0, ev, 1_000_000, 64), u)


def test_distinct_needs_enough_rows_and_ring_gate():
    with pytest.raises(ValueError):
        oracle.sample_distinct(2, 0, 0, 10, 11)
    r = oracle.Ring(50, 3, distinct=True)
    from inputs import experiences
    r.add(**experiences(20, state_dim=3))
    rc, _ = r.sample(1, 2, 0, 32)          # size 20 < B 32: not ready (Q29), nothing advances
    assert rc == oracle.NOT_READY and r.events == 0
    rc, b = r.sample(1, 2, 0, 20)          # B == size: a permutation of the ring
    assert rc == oracle.OK and sorted(b["idx"].tolist()) == list(range(20))
