"""Pins for oracle/cache.py and oracle/gather.py: SPEC worked examples
(S:199-201), brute-force degree order, shard bookkeeping."""
import numpy as np
import pytest

from oracle.cache import (POLICY_DEGREE, POLICY_NONE, access_counts, cache_capacity,
                          cache_slots, degree_rank)
from oracle.gather import gather_rows
from synth import chung_lu_graph, tiny_graph


def test_spec_cache_examples():
    g = tiny_graph("star10")
    slot, owner, _ = cache_slots(g.indptr, 0.0)
    assert (slot < 0).all()  # S:199 ratio 0 -> empty
    slot, _, _ = cache_slots(g.indptr, 1.0)
    assert (slot >= 0).all()  # S:200 ratio 1 -> all of V
    # capacity 1 -> {centre}; floor(r*11) = 1 for r = 1/11
    slot, _, _ = cache_slots(g.indptr, 1.0 / 11.0)
    assert cache_capacity(1.0 / 11.0, 11) == 1
    assert np.nonzero(slot >= 0)[0].tolist() == [0]


def test_spec_access_example():
    # resident {1,2}, batch {1,2} -> hits 2, misses 0
    slot = np.full(5, -1)
    slot[[1, 2]] = [0, 1]
    owner = np.where(slot >= 0, 0, -1)
    c = access_counts(slot, owner, np.array([1, 2]))
    assert c["hits"] == 2 and c["misses_host"] == 0
    c = access_counts(np.full(5, -1), np.full(5, -1), np.array([1, 2, 3]))
    assert c["hits"] == 0 and c["misses_host"] == 3  # policy none


def test_degree_rank_brute_force():
    indptr, _ = chung_lu_graph(500, 3000, 0.7, seed=4)
    deg = np.diff(indptr)
    order = sorted(range(500), key=lambda v: (-int(deg[v]), v))
    rank = degree_rank(indptr)
    assert [int(rank[v]) for v in order] == list(range(500))


def test_capacity_rounding_and_errors():
    assert cache_capacity(0.2, 2708) == 541  # floor(541.6)
    assert cache_capacity(0.5, 169343) == 84671
    assert cache_capacity(1.0, 7) == 7
    assert cache_capacity(0.7, 10, POLICY_NONE) == 0
    for r in (-0.1, 1.5, float("nan")):
        with pytest.raises(ValueError):
            cache_capacity(r, 10)


def test_hit_rate_monotone_in_ratio():
    indptr, _ = chung_lu_graph(2000, 16000, 0.5, seed=1)
    rows = np.random.default_rng(0).permutation(2000)[:700]
    prev = -1
    for r in (0.0, 0.1, 0.2, 0.5, 0.9, 1.0):
        slot, owner, _ = cache_slots(indptr, r)
        h = access_counts(slot, owner, rows)["hits"]
        assert h >= prev
        prev = h
    assert prev == 700


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_sharded_bookkeeping(G):
    indptr, _ = chung_lu_graph(1000, 6000, 0.5, seed=5)
    slot, owner, local = cache_slots(indptr, 0.37, world=G)
    cached = np.nonzero(slot >= 0)[0]
    assert cached.size == cache_capacity(0.37, 1000)
    pairs = set(zip(owner[cached].tolist(), local[cached].tolist()))
    assert len(pairs) == cached.size  # (owner, local) is a bijection onto the cache
    for o in range(G):
        loc = sorted(local[cached][owner[cached] == o].tolist())
        assert loc == list(range(len(loc)))  # shard o holds slots 0..len-1
    rows = np.arange(1000)
    for me in range(G):
        c = access_counts(slot, owner, rows, me)
        assert c["hits_local"] == int((owner == me).sum())
        assert c["hits_local"] + c["hits_peer"] + c["misses_host"] == 1000


def test_gather_bit_exact():
    rng = np.random.default_rng(2)
    feats = rng.standard_normal((50, 12)).astype(np.float32)
    rows = rng.integers(0, 50, size=30)
    X = gather_rows(feats, rows)
    for i, r in enumerate(rows):
        assert X[i].tobytes() == feats[r].tobytes()
