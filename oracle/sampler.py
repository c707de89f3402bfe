"""Node-wise fanout sampling and block construction (oracle side).

Paper: Eq.2 -- B^l = U_{v in B^{l-1}} u * 1_{p(eta)}(k^l / |N(v)|),
u in N(v); Algorithm 1 line 2 SubgraphSampling(G, B^0_i);
mini-batch subgraph G_i(V_i, E_i).

Readings:
  Q1  exact-k uniform sampling WITHOUT replacement; nodes with
      degree <= k take all neighbours.
  Q2  fanouts[0] applies to the seeds (hop 0).
  Q3  union frontiers: F_{h+1} = F_h ++ (new ids); every dst is re-expanded
      at the next hop with the hop-h key.
  Q4  Philox draws keyed by (rng_seed; hop, node, draw index); Floyd's
      algorithm turns k draws into a uniform k-subset of positions.
  Q5  sampled neighbours of a row in ascending CSR position.
  Q6  new local ids in first-appearance order of the (dst, position) scan,
      dst prefix kept (F_h occupies local ids 0..n_h-1).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np

from .philox import draw, uniform_int


def floyd_positions(d: int, k: int, ts: Sequence[int]) -> List[int]:
    """Floyd's algorithm for a k-subset of range(d), given the k integers
    t_s in [0, d-k+s] (s = 0..k-1).  Returns the positions ascending.

        S = {}
        for s in 0..k-1:  j = d-k+s;  S += {j} if t_s in S else {t_s}

    With exactly-uniform t_s every k-subset is produced by exactly k!
    tuples (pinned by exhaustive enumeration in the tests).
    """
    assert 0 < k <= d
    S: List[int] = []
    for s in range(k):
        j = d - k + s
        t = int(ts[s])
        assert 0 <= t <= j
        S.append(j if t in S else t)
    return sorted(S)


def sample_hop_positions(deg: np.ndarray, nodes: np.ndarray, k: int, hop: int,
                         rng_seed: int) -> List[np.ndarray]:
    """Per node: min(k, deg) distinct neighbour positions, ascending (Q1, Q4, Q5).

    Vectorised over nodes (independent problems); the loop over draw index s
    is Floyd's loop, in its order.
    """
    deg = np.asarray(deg, dtype=np.int64)
    nodes = np.asarray(nodes, dtype=np.int64)
    out: List[np.ndarray] = [None] * len(nodes)  # type: ignore
    small = np.nonzero(deg <= k)[0]
    for i in small:
        out[i] = np.arange(deg[i], dtype=np.int64)
    big = np.nonzero(deg > k)[0]
    if big.size:
        d = deg[big]
        v = nodes[big]
        sel = np.empty((big.size, k), dtype=np.int64)
        for s in range(k):
            j = d - k + s
            t = uniform_int(draw(rng_seed, hop, v, s), j).astype(np.int64)
            member = (sel[:, :s] == t[:, None]).any(axis=1) if s else np.zeros(big.size, bool)
            sel[:, s] = np.where(member, j, t)
        sel.sort(axis=1)
        for r, i in enumerate(big):
            out[i] = sel[r]
    return out


def locality_weight(bias: float) -> int:
    """Selection weight of a cached neighbour for locality bias b (NEXT-2):
    SPEC's p(eta) = 1 + 4 b eta (the paper says only that the
    probability is "a function of data locality").  Reading Q26:
    b is a multiple of 1/4, so the weight W = 1 + 4b is an integer in 1..5
    and the draw is exact integer arithmetic."""
    w = 1.0 + 4.0 * float(bias)
    if not (0.0 <= bias <= 1.0) or abs(w - round(w)) > 1e-12:
        raise ValueError("parameter error: locality bias must be in {0, 0.25, 0.5, 0.75, 1}")
    return int(round(w))


def successive_positions(d: int, k: int, cached: Sequence[bool], ts: Sequence[int], W: int) -> List[int]:
    """Weighted sampling without replacement, successive form (reading Q26):
    cached neighbours weigh W, the others 1; at draw s the remaining weight is
    T = W c + m (c cached, m uncached left) and the 32-bit draw u_s picks
    t = floor(u_s T / 2^32); t < W c selects the (t div W)-th remaining cached
    neighbour, else the (t - W c)-th remaining uncached one, "remaining" in
    ascending CSR position.  Positions returned ascending.  d <= k: all."""
    if d <= k:
        return list(range(d))
    cpos = [p for p in range(d) if cached[p]]
    upos = [p for p in range(d) if not cached[p]]
    taken = {0: [], 1: []}  # class -> ranks taken (sorted)
    lists = {0: cpos, 1: upos}
    out = []
    for s in range(k):
        c = len(cpos) - len(taken[0])
        m = len(upos) - len(taken[1])
        T = W * c + m
        t = (int(ts[s]) * T) >> 32
        if t < W * c:
            cls, j = 0, t // W
        else:
            cls, j = 1, t - W * c
        r = j
        for x in taken[cls]:  # j-th rank not yet taken
            if x <= r:
                r += 1
        taken[cls] = sorted(taken[cls] + [r])
        out.append(lists[cls][r])
    return sorted(out)


def sample_hop_positions_biased(indptr: np.ndarray, indices: np.ndarray, nodes: np.ndarray, k: int, hop: int,
                                rng_seed: int, cached_mask: np.ndarray, W: int) -> List[np.ndarray]:
    """Locality-biased node-wise sampling of one hop (NEXT-2, reading Q26):
    per node, the same Philox draws (rng_seed; hop, node, s) as the unbiased
    sampler, fed to successive_positions with cached_mask[neighbour]."""
    out = []
    for v in np.asarray(nodes, dtype=np.int64).tolist():
        b, e = int(indptr[v]), int(indptr[v + 1])
        d = e - b
        if d <= k:
            out.append(np.arange(d, dtype=np.int64))
            continue
        ts = [int(x) for x in draw(rng_seed, hop, np.full(k, v, dtype=np.int64), np.arange(k))]
        flags = cached_mask[np.asarray(indices[b:e], dtype=np.int64)]
        out.append(np.asarray(successive_positions(d, k, flags.tolist(), ts, W), dtype=np.int64))
    return out


@dataclasses.dataclass
class Block:
    """Sampled block b_h: dst = F_h (n_dst rows), src = F_{h+1} (n_src rows).

    indptr int64[n_dst+1]; indices int64[nnz] are LOCAL ids into F_{h+1};
    src_global = F_{h+1} (global ids, dst prefix first).
    """
    n_dst: int
    n_src: int
    indptr: np.ndarray
    indices: np.ndarray
    src_global: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])

    def counts(self) -> np.ndarray:
        return np.diff(self.indptr)


def relabel(frontier: np.ndarray, rows: List[np.ndarray]):
    """First-appearance relabelling (Q6), written as the plain scan.

    Returns (F_next global ids, block indptr, block indices local)."""
    local = {}
    F_next = []
    for i, g in enumerate(frontier.tolist()):
        local[g] = i
        F_next.append(g)
    indices = []
    indptr = [0]
    for row in rows:
        for u in row.tolist():
            lid = local.get(u)
            if lid is None:
                lid = len(F_next)
                local[u] = lid
                F_next.append(u)
            indices.append(lid)
        indptr.append(len(indices))
    return (np.asarray(F_next, dtype=np.int64), np.asarray(indptr, dtype=np.int64),
            np.asarray(indices, dtype=np.int64))


def sample_blocks(indptr: np.ndarray, indices: np.ndarray, seeds: Sequence[int],
                  fanouts: Sequence[int], rng_seed: int, cached_mask: Optional[np.ndarray] = None,
                  locality_bias: float = 0.0):
    """SubgraphSampling (Algorithm 1 line 2) for L = len(fanouts) hops.

    Returns (frontiers [F_0..F_L], blocks [b_0..b_{L-1}]).
    Preconditions (SPEC S:114 parameter errors): seeds non-empty, unique,
    in range; every fanout >= 1.
    """
    seeds = np.asarray(seeds, dtype=np.int64)
    n = len(indptr) - 1
    if seeds.size < 1 or len(fanouts) < 1 or min(fanouts) < 1:
        raise ValueError("parameter error")
    if seeds.min() < 0 or seeds.max() >= n or np.unique(seeds).size != seeds.size:
        raise ValueError("parameter error: seeds must be unique ids in [0, N)")
    deg_all = np.diff(np.asarray(indptr, dtype=np.int64))
    F = seeds
    frontiers = [F]
    blocks = []
    W = locality_weight(locality_bias)
    for h, k in enumerate(fanouts):
        if W > 1:  # NEXT-2: locality-biased (cached neighbours weigh W)
            pos = sample_hop_positions_biased(indptr, indices, F, int(k), h, rng_seed, cached_mask, W)
        else:
            pos = sample_hop_positions(deg_all[F], F, int(k), h, rng_seed)
        rows = [np.asarray(indices[indptr[v] + p], dtype=np.int64) for v, p in zip(F.tolist(), pos)]
        F_next, bptr, bidx = relabel(F, rows)
        blocks.append(Block(n_dst=len(F), n_src=len(F_next), indptr=bptr, indices=bidx,
                            src_global=F_next))
        F = F_next
        frontiers.append(F)
    return frontiers, blocks
