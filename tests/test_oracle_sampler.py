"""Pins for oracle/sampler.py: Floyd exhaustive enumeration, SPEC worked
examples, soundness properties, networkx BFS for exhaustive fanout, Eq.12
bound, relabel order, rank independence."""
import itertools
import math
from collections import Counter

import networkx as nx
import numpy as np
import pytest

from oracle.philox import draw, uniform_int
from oracle.sampler import floyd_positions, relabel, sample_blocks, sample_hop_positions
from synth import chung_lu_graph, tiny_graph


@pytest.mark.parametrize("d,k", [(2, 1), (3, 2), (4, 2), (5, 2), (5, 3), (6, 3), (6, 4), (7, 5)])
def test_floyd_exhaustive_uniform(d, k):
    """Every draw tuple (t_s in [0, d-k+s]) -> each k-subset exactly k! times."""
    ranges = [range(d - k + s + 1) for s in range(k)]
    cnt = Counter(tuple(floyd_positions(d, k, ts)) for ts in itertools.product(*ranges))
    assert len(cnt) == math.comb(d, k)
    assert set(cnt.values()) == {math.factorial(k)}
    for subset in cnt:
        assert len(set(subset)) == k and all(0 <= p < d for p in subset)


def test_vectorised_hop_matches_scalar_floyd():
    rng = np.random.default_rng(5)
    deg = rng.integers(0, 40, size=500)
    nodes = rng.permutation(10**6)[:500]
    seed = 0xABCDEF
    for k in (1, 3, 5, 10, 15, 25):
        got = sample_hop_positions(deg, nodes, k, 2, seed)
        for d, v, g in zip(deg, nodes, got):
            if d <= k:
                assert g.tolist() == list(range(d))
            else:
                ts = [int(uniform_int(draw(seed, 2, v, s), d - k + s)) for s in range(k)]
                assert g.tolist() == floyd_positions(int(d), k, ts)


def test_floyd_philox_chi_square():
    """Statistical pin with the real draws: d=6,k=3 over 40000 nodes."""
    n = 40000
    deg = np.full(n, 6)
    pos = sample_hop_positions(deg, np.arange(n), 3, 0, 77)
    cnt = Counter(tuple(p.tolist()) for p in pos)
    assert len(cnt) == 20
    exp = n / 20
    chi2 = sum((c - exp) ** 2 / exp for c in cnt.values())
    assert chi2 < 43.8  # 19 dof, p = 0.001


def _edge_set(g):
    s = set()
    for v in range(g.n):
        for u in g.indices[g.indptr[v]:g.indptr[v + 1]]:
            s.add((v, int(u)))
    return s


def test_spec_path_example():
    g = tiny_graph("path5")
    for seed in range(5):
        F, blocks = sample_blocks(g.indptr, g.indices, [2], [2], seed)
        assert sorted(F[-1].tolist()) == [1, 2, 3]


def test_spec_star_example():
    g = tiny_graph("star10")
    for seed in range(20):
        F, blocks = sample_blocks(g.indptr, g.indices, [0], [3], seed)
        assert len(F[-1]) == 4


def test_soundness_random_graphs():
    rng = np.random.default_rng(3)
    for trial in range(30):
        n = int(rng.integers(20, 300))
        nnz = 2 * int(rng.integers(n, 4 * n))
        indptr, indices = chung_lu_graph(n, nnz, 0.6, seed=trial)
        deg = np.diff(indptr)
        seeds = rng.permutation(n)[: int(rng.integers(1, 20))]
        fan = [int(x) for x in rng.integers(1, 8, size=int(rng.integers(1, 4)))]
        F, blocks = sample_blocks(indptr, indices, seeds, fan, int(rng.integers(0, 2**63)))
        assert F[0].tolist() == seeds.tolist()
        for h, b in enumerate(blocks):
            assert b.n_dst == len(F[h]) and b.n_src == len(F[h + 1])
            assert F[h + 1][: b.n_dst].tolist() == F[h].tolist()  # dst prefix (Q3, Q6)
            assert len(set(F[h + 1].tolist())) == b.n_src  # bijection
            assert b.n_src <= b.n_dst * (1 + fan[h])  # Eq.12 / S:106 bound
            for r in range(b.n_dst):
                v = int(F[h][r])
                nb = b.indices[b.indptr[r]:b.indptr[r + 1]]
                glob = F[h + 1][nb]
                row = set(indices[indptr[v]:indptr[v + 1]].tolist())
                assert len(nb) == min(fan[h], deg[v])  # exact-k, d<=k takes all
                assert len(set(glob.tolist())) == len(nb)  # no duplicates
                assert set(glob.tolist()) <= row  # every sampled edge exists
                # ascending CSR position (Q5): neighbour ids are sorted in CSR rows
                assert list(glob) == sorted(glob)


def test_exhaustive_fanout_equals_bfs_ball():
    """k >= max degree gives exactly the L-hop neighbourhood."""
    indptr, indices = chung_lu_graph(400, 1600, 0.5, seed=9)
    G = nx.Graph()
    G.add_nodes_from(range(400))
    for v in range(400):
        for u in indices[indptr[v]:indptr[v + 1]]:
            G.add_edge(v, int(u))
    kmax = int(np.diff(indptr).max())
    seeds = [3, 77, 150]
    for L in (1, 2, 3):
        F, _ = sample_blocks(indptr, indices, seeds, [kmax] * L, 1234)
        ball = set()
        for s in seeds:
            ball |= set(nx.single_source_shortest_path_length(G, s, cutoff=L))
        assert set(F[-1].tolist()) == ball


def test_relabel_first_appearance_order():
    # independent statement: new ids follow the order of first occurrence
    rng = np.random.default_rng(0)
    frontier = np.array([10, 20, 30])
    rows = [rng.integers(0, 50, size=int(rng.integers(0, 6))) for _ in range(3)]
    F, ptr, idx = relabel(frontier, rows)
    flat = np.concatenate(rows) if rows else np.array([])
    new = [u for u in dict.fromkeys(flat.tolist()) if u not in (10, 20, 30)]
    assert F.tolist() == [10, 20, 30] + new
    assert (F[idx] == flat).all()


def test_rank_independence():
    """Sampling is keyed by node: a node's sampled neighbours do not depend on
    which other seeds share its batch (multi-GPU invariant)."""
    indptr, indices = chung_lu_graph(3000, 30000, 0.5, seed=2)
    seeds = np.random.default_rng(1).permutation(3000)[:64]
    fan = [6, 4]
    Fa, Ba = sample_blocks(indptr, indices, seeds, fan, 99)
    Fb, Bb = sample_blocks(indptr, indices, seeds[:32], fan, 99)

    def neigh(F, B):
        out = {}
        for h, b in enumerate(B):
            for r in range(b.n_dst):
                out[(h, int(F[h][r]))] = sorted(F[h + 1][b.indices[b.indptr[r]:b.indptr[r + 1]]].tolist())
        return out

    na, nb = neigh(Fa, Ba), neigh(Fb, Bb)
    for key, val in nb.items():
        assert na[key] == val


def test_parameter_errors():
    g = tiny_graph("path5")
    for seeds, fan in [([], [2]), ([0, 0], [2]), ([5], [2]), ([1], [0]), ([1], [])]:
        with pytest.raises(ValueError):
            sample_blocks(g.indptr, g.indices, seeds, fan, 0)
