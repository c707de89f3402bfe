"""Synthetic power-law graphs shaped like the paper's datasets (seeded).

Recipe:
  * Chung-Lu, undirected.  Expected-degree weights w_i ∝ (i+1)^-beta.  Both
    endpoints of each candidate edge are drawn ∝ w by inverse CDF with a
    numpy PCG64 generator keyed by `graph_seed`.  Self-loops and duplicate
    pairs are dropped and the draw is topped up until exactly nnz/2
    undirected edges exist (surplus candidates are discarded by a seeded
    choice).  The graph is symmetrised, vertex ids are randomly permuted (so
    degree order is not id order) and every CSR row is sorted by id.
    PAPER.md §4.1 P:433 ("power-law graphs" for data enhancement);
    SPEC.md S:36-44 (generate_power_law), S:72 (symmetrise).
  * CSR nnz equals the stated edge count of the dataset (reading Q14).
  * Features fp32 N(0,1), stored with the row stride padded to
    a multiple of 4 floats (reading Q16); padding columns are zero.
  * Labels uniform in [0, C).
  * Initial weights uniform(+-1/sqrt(fan_in)) (reading Q12), generated here
    and passed in to both sides as inputs.

Nothing in this module samples neighbours, relabels, caches or computes a
GNN layer.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np

GRAPH_SEED = 0
FEAT_SEED = 1
LABEL_SEED = 2
EPOCH_SEED0 = 3
INIT_SEED = 4
BASE_RNG_SEED = 0x5EED


def row_stride(d: int) -> int:
    """Stored row stride (floats) for logical width d: next multiple of 4."""
    return (int(d) + 3) & ~3


# BASELINE.json "configs", made concrete as in SURVEY §8(d).
CONFIGS: Dict[str, dict] = {
    "cora": dict(name="cora", n=2708, nnz=10556, d=1433, C=7, fanouts=[10, 5],
                 batch=64, ratio=0.2, beta=0.45, hidden=256),
    "arxiv": dict(name="arxiv", n=169343, nnz=1166243 - 1166243 % 2, d=128, C=40,
                  fanouts=[15, 10, 5], batch=1024, ratio=0.5, beta=0.5, hidden=256),
    "reddit": dict(name="reddit", n=232965, nnz=114615892, d=602, C=41, fanouts=[25, 10],
                   batch=1024, ratio=0.1, beta=0.25, hidden=256),
    "products": dict(name="products", n=2449029, nnz=61859140, d=100, C=47,
                     fanouts=[15, 10, 5], batch=4096, ratio=1.0, beta=0.5, hidden=256),
    "papers100m": dict(name="papers100m", n=111059956, nnz=1615685872, d=128, C=172,
                       fanouts=[15, 10, 5], batch=8192, ratio=1.0, beta=0.5, hidden=256),
    # products with 128-d features (512-byte rows): a layout experiment
    # (DESIGN.md §9), not a BASELINE config
    "products_d128": dict(name="products_d128", n=2449029, nnz=61859140, d=128, C=47,
                          fanouts=[15, 10, 5], batch=4096, ratio=1.0, beta=0.5, hidden=256),
    # small config used by unit/parity tests: several tiles and a ragged tail
    "mini": dict(name="mini", n=20000, nnz=200000, d=100, C=47, fanouts=[15, 10, 5],
                 batch=512, ratio=0.3, beta=0.5, hidden=64),
}


@dataclasses.dataclass
class GraphData:
    """CSR graph + host features/labels.  indptr int64[n+1], indices int32[nnz]."""

    n: int
    indptr: np.ndarray
    indices: np.ndarray
    feats: np.ndarray  # float32 [n, stride]; columns >= d are zero
    d: int
    labels: np.ndarray  # int32 [n]
    C: int
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])

    @property
    def stride(self) -> int:
        return int(self.feats.shape[1])

    def degree(self) -> np.ndarray:
        return np.diff(self.indptr)


def csr_from_edges(n: int, src: np.ndarray, dst: np.ndarray):
    """Directed edge list -> CSR (rows sorted by neighbour id, duplicates kept)."""
    key = np.asarray(src, dtype=np.int64) * np.int64(n)
    key += np.asarray(dst, dtype=np.int64)
    return csr_from_keys(n, key)


def csr_from_keys(n: int, key: np.ndarray):
    """CSR from packed directed edge keys src*n + dst (sorted in place)."""
    key.sort()
    rows = key // n
    cols = (key - rows * n).astype(np.int32)
    del key
    counts = np.bincount(rows, minlength=n).astype(np.int64)
    del rows
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return indptr, cols


_U_BITS = 38  # resolution of the uniform draws (2^-38, far below the smallest cdf step)
_IDX_BITS = 25
_IDX_MASK = (1 << _IDX_BITS) - 1


def _inverse_cdf(cdf: np.ndarray, rng: np.random.Generator, count: int) -> np.ndarray:
    """count draws of an index i with P(i) = cdf[i] - cdf[i-1].

    u = U38 / 2^38 with U38 uniform 38-bit integers; the queries are sorted
    (packed with their position into one int64 key, a fast integer sort) so
    that searchsorted walks the cdf sequentially."""
    assert count <= _IDX_MASK
    u = rng.integers(0, 1 << _U_BITS, size=count, dtype=np.int64)
    key = (u << _IDX_BITS) | np.arange(count, dtype=np.int64)
    key.sort()
    pos = key & _IDX_MASK
    us = (key >> _IDX_BITS).astype(np.float64) * (1.0 / (1 << _U_BITS))
    out = np.empty(count, dtype=np.int64)
    out[pos] = np.searchsorted(cdf, us, side="right")
    return out


def _sorted_unique(k: np.ndarray) -> np.ndarray:
    k = np.sort(k)
    if k.size == 0:
        return k
    keep = np.empty(k.size, dtype=bool)
    keep[0] = True
    np.not_equal(k[1:], k[:-1], out=keep[1:])
    return k[keep]


def _chung_lu_keys_large(n: int, m: int, cdf: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    """The same edge draws for m beyond one draw batch (papers100M-sized):
    candidates are drawn in batches of at most _IDX_MASK and de-duplicated
    with ONE sort over all of them, instead of a sort per batch; the caller's
    loop then tops up any shortfall."""
    chunks = []
    total = int(m * 1.05) + 64
    done = 0
    while done < total:
        batch = min(total - done, _IDX_MASK)
        a = _inverse_cdf(cdf, rng, batch)
        b = _inverse_cdf(cdf, rng, batch)
        np.minimum(a, n - 1, out=a)
        np.minimum(b, n - 1, out=b)
        lo = np.minimum(a, b)
        hi = np.maximum(a, b)
        del a, b
        ok = lo != hi
        chunks.append(lo[ok] * np.int64(n) + hi[ok])
        del lo, hi, ok
        done += batch
    keys = np.concatenate(chunks)
    del chunks
    return _sorted_unique(keys)


def chung_lu_graph(n: int, nnz: int, beta: float, seed: int = GRAPH_SEED):
    """Undirected simple Chung-Lu graph with exactly nnz (even) CSR entries."""
    if nnz % 2:
        raise ValueError("nnz must be even for a symmetric graph")
    m = nnz // 2
    if m > n * (n - 1) // 2:
        raise ValueError("too many edges for a simple graph")
    rng = np.random.Generator(np.random.PCG64(seed))
    w = np.arange(1, n + 1, dtype=np.float64) ** (-float(beta))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    del w
    if m > _IDX_MASK:
        keys = _chung_lu_keys_large(n, m, cdf, rng)
    else:
        keys = np.empty(0, dtype=np.int64)
    while keys.shape[0] < m:
        need = m - keys.shape[0]
        batch = min(int(need * 1.05) + 64, _IDX_MASK)
        a = _inverse_cdf(cdf, rng, batch)
        b = _inverse_cdf(cdf, rng, batch)
        np.minimum(a, n - 1, out=a)
        np.minimum(b, n - 1, out=b)
        lo = np.minimum(a, b)
        hi = np.maximum(a, b)
        ok = lo != hi
        k = lo[ok] * np.int64(n) + hi[ok]
        keys = _sorted_unique(np.concatenate([keys, k]))
    if keys.shape[0] > m:
        keep = rng.choice(keys.shape[0], m, replace=False)
        keys = keys[np.sort(keep)]
    lo = keys // n
    hi = keys - lo * n
    del keys
    perm = rng.permutation(n).astype(np.int64)
    lo = perm[lo]
    hi = perm[hi]
    del perm
    key = np.concatenate([lo * np.int64(n) + hi, hi * np.int64(n) + lo])
    del lo, hi
    return csr_from_keys(n, key)


def make_features(n: int, d: int, seed: int = FEAT_SEED, stride: Optional[int] = None) -> np.ndarray:
    stride = row_stride(d) if stride is None else int(stride)
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.zeros((n, stride), dtype=np.float32)
    chunk = max(1, (1 << 24) // max(d, 1))
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        out[s:e, :d] = rng.standard_normal((e - s, d), dtype=np.float32)
    return out


def make_labels(n: int, C: int, seed: int = LABEL_SEED) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, C, size=n, dtype=np.int32)


def make_graph(cfg, graph_seed: int = GRAPH_SEED, with_feats: bool = True) -> GraphData:
    """Build the synthetic graph for a config name or dict."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n, nnz = int(cfg["n"]), int(cfg["nnz"])
    indptr, indices = chung_lu_graph(n, nnz, float(cfg["beta"]), graph_seed)
    d = int(cfg["d"])
    feats = make_features(n, d) if with_feats else np.zeros((0, row_stride(d)), np.float32)
    labels = make_labels(n, int(cfg["C"]))
    return GraphData(n=n, indptr=indptr, indices=indices, feats=feats, d=d,
                     labels=labels, C=int(cfg["C"]), name=cfg.get("name", ""))


def tiny_graph(kind: str, d: int = 4, C: int = 3, n: int = 0) -> GraphData:
    """Hand graphs for worked examples.

    kinds: path5 (0-1-2-3-4), star10 (K1,10, centre 0), clique<n>, isolated
    (path5 plus an isolated vertex 5), twostar (two K1,3 sharing nothing).
    """
    edges: List[Sequence[int]]
    if kind == "path5":
        nv, edges = 5, [(0, 1), (1, 2), (2, 3), (3, 4)]
    elif kind == "star10":
        nv, edges = 11, [(0, i) for i in range(1, 11)]
    elif kind == "clique":
        nv = n or 6
        edges = [(i, j) for i in range(nv) for j in range(i + 1, nv)]
    elif kind == "isolated":
        nv, edges = 6, [(0, 1), (1, 2), (2, 3), (3, 4)]
    elif kind == "twostar":
        nv, edges = 8, [(0, 1), (0, 2), (0, 3), (4, 5), (4, 6), (4, 7)]
    else:
        raise ValueError(kind)
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    src = np.concatenate([e[:, 0], e[:, 1]])
    dst = np.concatenate([e[:, 1], e[:, 0]])
    indptr, indices = csr_from_edges(nv, src, dst)
    feats = make_features(nv, d)
    labels = make_labels(nv, C)
    return GraphData(n=nv, indptr=indptr, indices=indices, feats=feats, d=d,
                     labels=labels, C=C, name=kind)


def epoch_seeds(n: int, epoch: int = 0) -> np.ndarray:
    """Seed order for one epoch (reading Q10): PCG64(EPOCH_SEED0+epoch).permutation(n)."""
    rng = np.random.Generator(np.random.PCG64(EPOCH_SEED0 + int(epoch)))
    return rng.permutation(n).astype(np.int32)


def init_weights(dims: Sequence[int], kind: str = "sage", seed: int = INIT_SEED):
    """Initial weights per layer: W [(2 if sage else 1)*d_in, d_out], b [d_out].

    uniform(+-1/sqrt(fan_in)) with fan_in = rows of W (reading Q12).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for i in range(len(dims) - 1):
        d_in, d_out = int(dims[i]), int(dims[i + 1])
        rows = 2 * d_in if kind == "sage" else d_in
        bound = 1.0 / np.sqrt(rows)
        W = rng.uniform(-bound, bound, size=(rows, d_out)).astype(np.float32)
        b = rng.uniform(-bound, bound, size=(d_out,)).astype(np.float32)
        out.append((W, b))
    return out
