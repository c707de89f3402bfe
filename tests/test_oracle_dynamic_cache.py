"""Pins of the dynamic (FIFO / LRU) cache oracle (NEXT-3, reading Q27):
SPEC's worked example, hand-simulated FIFO vs LRU sequences, and
the invariants of S:213-217 (capacity never exceeded, replaced <= misses,
ratio 1 => everything hits once seen)."""
import numpy as np
import pytest

from oracle.cache import POLICY_FIFO, POLICY_LRU, DynamicCache


def test_spec_fifo_example():
    # capacity 2, FIFO, empty start; batches {1,2}, {3}, {1}: admitting 3
    # evicts 1, so the third batch misses
    c = DynamicCache(10, 2, POLICY_FIFO)
    assert c.access_batch([1, 2]) == dict(rows=2, hits=0, misses=2, replaced=0)
    assert c.access_batch([3]) == dict(rows=1, hits=0, misses=1, replaced=1)
    assert c.resident() == {2, 3}
    assert c.access_batch([1])["misses"] == 1


def test_fifo_vs_lru_hand_simulated():
    # capacity 2: {1,2} {1} {3} -- FIFO evicts 1 (oldest admission),
    # LRU evicts 2 (1 was used more recently)
    f = DynamicCache(10, 2, POLICY_FIFO)
    lru = DynamicCache(10, 2, POLICY_LRU)
    for c in (f, lru):
        c.access_batch([1, 2])
        assert c.access_batch([1])["hits"] == 1
        c.access_batch([3])
    assert f.resident() == {2, 3}
    assert lru.resident() == {1, 3}


def test_batch_larger_than_capacity():
    # 5 misses into capacity 2: the last two admitted stay, 3 in-batch
    # evictions (replaced counts every eviction, <= misses)
    c = DynamicCache(10, 2, POLICY_LRU)
    out = c.access_batch([5, 6, 7, 8, 9])
    assert out == dict(rows=5, hits=0, misses=5, replaced=3)
    assert c.resident() == {8, 9}


def test_lru_hits_evicted_before_newer_admissions():
    # capacity 3: {1,2,3}; then batch {3, 4, 5, 6}: 3 is a hit (stamp 1);
    # 4 evicts 1, 5 evicts 2 (stamp 0), 6 evicts 3 (stamp 1, seq 2 < 4's)
    c = DynamicCache(10, 3, POLICY_LRU)
    c.access_batch([1, 2, 3])
    out = c.access_batch([3, 4, 5, 6])
    assert out == dict(rows=4, hits=1, misses=3, replaced=3)
    assert c.resident() == {4, 5, 6}


@pytest.mark.parametrize("policy", [POLICY_FIFO, POLICY_LRU])
def test_invariants_random_batches(policy):
    rng = np.random.default_rng(1)
    n, C = 200, 37
    c = DynamicCache(n, C, policy)
    for t in range(60):
        rows = rng.choice(n, rng.integers(1, 80), replace=False)
        out = c.access_batch(rows)
        assert out["replaced"] <= out["misses"]
        assert len(c.resident()) <= C
        res = c.resident()
        assert all(c.slot[v] >= 0 for v in res)
        assert int((c.slot >= 0).sum()) == len(res)  # slot map and owners agree
        assert out["hits"] + out["misses"] == len(rows)


@pytest.mark.parametrize("policy", [POLICY_FIFO, POLICY_LRU])
def test_full_capacity_second_epoch_all_hits(policy):
    n = 50
    c = DynamicCache(n, n, policy)
    perm = np.random.default_rng(2).permutation(n)
    for i in range(0, n, 8):
        c.access_batch(perm[i:i + 8])
    hits = sum(c.access_batch(perm[i:i + 8])["hits"] for i in range(0, n, 8))
    assert hits == n and c.replaced == 0


def test_zero_capacity_never_hits():
    c = DynamicCache(10, 0, POLICY_LRU)
    assert c.access_batch([1, 2])["hits"] == 0 and c.access_batch([1])["hits"] == 0
