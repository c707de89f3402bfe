"""Pins of the locality-biased sampler (NEXT-2, reading Q26) on the CPU.

The weight rule (cached neighbours weigh W = 1 + 4b, others 1; SPEC S:123,
S:159) is pinned against the closed-form law of successive weighted
sampling without replacement, P(a then b) = w_a/S * w_b/(S - w_a), by
EXACT enumeration of the multiply-high draw map (each t in [0, T) is hit by
ceil((t+1) 2^32 / T) - ceil(t 2^32 / T) of the 2^32 draws), plus a
statistical check with the real Philox draws, the SPEC's bias-monotonicity
property and the sampler invariants.
"""
import itertools
import math

import numpy as np
import pytest

from oracle.cache import cache_slots
from oracle.philox import draw
from oracle.sampler import locality_weight, sample_blocks, successive_positions

TWO32 = 1 << 32


def _rep(t, T):
    """A 32-bit draw that the multiply-high map sends to t, and the exact
    probability of t."""
    lo = -(-t * TWO32 // T)
    hi = -(-(t + 1) * TWO32 // T)
    return lo, (hi - lo) / TWO32


def _exact_law(d, k, cached, W):
    """{sorted subset: probability} of successive_positions over all draws."""
    law = {}

    def rec(ts, prob):
        s = len(ts)
        if s == k:
            key = tuple(successive_positions(d, k, cached, ts, W))
            law[key] = law.get(key, 0.0) + prob
            return
        picked = successive_positions(d, s, cached, ts, W) if s else []
        c = sum(1 for p in range(d) if cached[p]) - sum(1 for p in picked if cached[p])
        m = (d - sum(cached)) - sum(1 for p in picked if not cached[p])
        T = W * c + m
        for t in range(T):
            u, pt = _rep(t, T)
            rec(ts + [u], prob * pt)

    rec([], 1.0)
    return law


def _closed_form(d, k, cached, W):
    w = [W if cached[p] else 1 for p in range(d)]
    law = {}
    for order in itertools.permutations(range(d), k):
        p, S = 1.0, float(sum(w))
        for x in order:
            p *= w[x] / S
            S -= w[x]
        key = tuple(sorted(order))
        law[key] = law.get(key, 0.0) + p
    return law


@pytest.mark.parametrize("d,k,cached,W", [
    (5, 2, [1, 0, 0, 1, 0], 2),
    (5, 2, [1, 0, 0, 1, 0], 5),
    (6, 3, [0, 1, 1, 0, 0, 1], 3),
    (4, 3, [1, 1, 1, 1], 5),  # all cached: uniform
    (5, 3, [0, 0, 0, 0, 0], 4),  # none cached: uniform
    (5, 2, [1, 0, 0, 1, 0], 1),  # W = 1: uniform without replacement
])
def test_successive_law_exact(d, k, cached, W):
    got = _exact_law(d, k, cached, W)
    want = _closed_form(d, k, cached, W)
    assert set(got) == set(want)
    for key in want:
        assert abs(got[key] - want[key]) < 1e-8, (key, got[key], want[key])


def test_successive_law_with_philox_draws():
    d, k, W = 7, 3, 5
    cached = [1, 0, 0, 1, 0, 0, 0]
    want = _closed_form(d, k, cached, W)
    n = 40000
    counts = {}
    ts = [draw(0x5EED, 1, np.arange(n, dtype=np.int64), s) for s in range(k)]
    for v in range(n):
        key = tuple(successive_positions(d, k, cached, [int(ts[s][v]) for s in range(k)], W))
        counts[key] = counts.get(key, 0) + 1
    chi2 = sum((counts.get(key, 0) - n * p) ** 2 / (n * p) for key, p in want.items())
    dof = len(want) - 1
    assert chi2 < dof + 5 * math.sqrt(2 * dof), chi2  # ~5 sigma


def test_locality_weight_grid():
    assert [locality_weight(b) for b in (0, 0.25, 0.5, 0.75, 1.0)] == [1, 2, 3, 4, 5]
    for bad in (-0.25, 0.3, 1.25):
        with pytest.raises(ValueError):
            locality_weight(bad)


@pytest.fixture(scope="module")
def mini_graph():
    from synth import make_graph

    return make_graph("mini", with_feats=False)


def test_biased_invariants_and_monotone_hit_fraction(mini_graph):
    gd = mini_graph
    slot, _, _ = cache_slots(gd.indptr, 0.2)
    cached = slot >= 0
    rng = np.random.default_rng(5)
    frac = []
    for bias in (0.0, 0.5, 1.0):
        fr = []
        for rep in range(6):
            seeds = rng.choice(gd.n, 64, replace=False)
            F, blocks = sample_blocks(gd.indptr, gd.indices, seeds, [10, 5], 100 + rep, cached, bias)
            for h, b in enumerate(blocks):  # invariants: true neighbours, distinct, min(k, deg)
                k = [10, 5][h]
                for r in range(b.n_dst):
                    v = int(F[h][r])
                    nb = b.src_global[b.indices[b.indptr[r]:b.indptr[r + 1]]]
                    adj = set(gd.indices[gd.indptr[v]:gd.indptr[v + 1]].tolist())
                    assert len(set(nb.tolist())) == len(nb) == min(k, len(adj))
                    assert set(nb.tolist()) <= adj
            fr.append(cached[F[-1]].mean())
        frac.append((np.mean(fr), np.std(fr) / np.sqrt(len(fr))))
    # the cached fraction of V_i does not decrease with the bias
    for (m0, e0), (m1, e1) in zip(frac, frac[1:]):
        assert m1 >= m0 - max(e0, e1), frac
    assert frac[-1][0] > frac[0][0]


def test_bias_zero_is_the_unbiased_sampler(mini_graph):
    gd = mini_graph
    slot, _, _ = cache_slots(gd.indptr, 0.2)
    seeds = np.arange(0, 2000, 37)
    a = sample_blocks(gd.indptr, gd.indices, seeds, [5, 3], 9)
    b = sample_blocks(gd.indptr, gd.indices, seeds, [5, 3], 9, slot >= 0, 0.0)
    for x, y in zip(a[1], b[1]):
        assert (x.indices == y.indices).all() and (x.indptr == y.indptr).all()
