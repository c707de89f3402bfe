"""Aggregate / Combine, loss, backward and SGD for sampled blocks (oracle side).

Paper: Eq.1
    a_v^l = Aggregate^l(h_u^{l-1} | u in N(v) U h_v^{l-1}),  h_v^l = Combine^l(a_v^l)
Algorithm 1 lines 4-8: Aggregate, Combine, LossFunction,
Backwards; plain gradient descent.

Readings:
  Q11 SAGE (default): h_v = act(h_v W_s + a_v W_n + b), a_v = mean (or sum)
      of the sampled neighbours' h_u; GCN: h_v = act(a'_v W + b),
      a'_v = (h_v + sum_u h_u)/(c_v+1) (or the plain sum).  act = ReLU
      except the last layer.  Edge features unused.
  Q13 one loss and one backward per iteration, after layer L.
  Q15 a row with c_v = 0 aggregates to 0 (SAGE); GCN keeps h_v.
  Loss: (1/B_global) sum_i [logsumexp(z_i) - z_i[y_i]]; gradients scaled by
  1/B_global so that the sum over ranks equals the concatenated-batch
  gradient.

All arithmetic in float64.  Library primitives used as steps: scipy.sparse
matrix products (the aggregation operator P), numpy matmul.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import numpy as np
import scipy.sparse as sp

from .sampler import Block, sample_blocks


def agg_matrix(block: Block, kind: str = "sage", aggr: str = "mean") -> sp.csr_matrix:
    """Aggregation operator P (n_dst x n_src) so that A = P @ H_src.

    sage/mean: P[v,u] = 1/c_v;  sage/sum: 1;
    gcn/mean:  P[v,u] = P[v,v] = 1/(c_v+1);  gcn/sum: 1 (self included).
    """
    c = block.counts().astype(np.float64)
    rows = np.repeat(np.arange(block.n_dst), block.counts())
    cols = np.asarray(block.indices, dtype=np.int64)
    if kind == "sage":
        w = (1.0 / c[rows]) if aggr == "mean" else np.ones(rows.size)
    elif kind == "gcn":
        w = (1.0 / (c[rows] + 1.0)) if aggr == "mean" else np.ones(rows.size)
        self_w = (1.0 / (c + 1.0)) if aggr == "mean" else np.ones(block.n_dst)
        rows = np.concatenate([rows, np.arange(block.n_dst)])
        cols = np.concatenate([cols, np.arange(block.n_dst)])
        w = np.concatenate([w, self_w])
    else:
        raise ValueError(kind)
    return sp.csr_matrix((w, (rows, cols)), shape=(block.n_dst, block.n_src))


def layer_fwd(block: Block, H_src: np.ndarray, W: np.ndarray, b: np.ndarray,
              relu: bool, kind: str = "sage", aggr: str = "mean", absval: bool = False):
    """One layer.  Returns (H_out [n_dst, d_out], A [n_dst, d_in]).

    absval=True evaluates the same expression on |.| of every operand: the
    magnitude bound used by the condition-aware tolerance (reading Q17)."""
    H = np.asarray(H_src, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    P = agg_matrix(block, kind, aggr)
    if absval:
        H, W, b = np.abs(H), np.abs(W), np.abs(b)
        P = abs(P)
    d_in = H.shape[1]
    A = P @ H
    if kind == "sage":
        Z = H[: block.n_dst] @ W[:d_in] + A @ W[d_in:] + b
    else:
        Z = A @ W + b
    Hout = np.maximum(Z, 0.0) if (relu and not absval) else Z
    return Hout, A


def ce_loss(z: np.ndarray, y: np.ndarray, n_global: int):
    """Softmax cross-entropy over the rank's seeds.
    Returns (loss, dz) with loss = (1/n_global) sum_i [lse(z_i) - z_i[y_i]]."""
    z = np.asarray(z, dtype=np.float64)
    y = np.asarray(y, dtype=np.int64)
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    se = e.sum(axis=1, keepdims=True)
    lse = (m + np.log(se))[:, 0]
    loss = float((lse - z[np.arange(z.shape[0]), y]).sum() / n_global)
    dz = e / se
    dz[np.arange(z.shape[0]), y] -= 1.0
    return loss, dz / n_global


def layer_bwd(block: Block, H_src: np.ndarray, A: np.ndarray, H_out: np.ndarray,
              W: np.ndarray, G: np.ndarray, relu: bool, need_dx: bool,
              kind: str = "sage", aggr: str = "mean"):
    """Backward of layer_fwd given G = dL/dH_out (post-activation).

    Returns (dW, db, dH_src or None):
      G' = G * 1[H_out > 0] (ReLU);  dW_s = H_dst^T G', dW_n = A^T G', db = sum G'
      dH_src = P^T (G' W_n^T) + [G' W_s^T ; 0]      (SAGE)
      dW = A'^T G', dH_src = P^T (G' W^T)            (GCN)
    """
    H = np.asarray(H_src, dtype=np.float64)
    A = np.asarray(A, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    G = np.asarray(G, dtype=np.float64)
    if relu:
        G = G * (np.asarray(H_out) > 0)
    d_in = H.shape[1]
    db = G.sum(axis=0)
    P = agg_matrix(block, kind, aggr)
    dX = None
    if kind == "sage":
        dW = np.concatenate([H[: block.n_dst].T @ G, A.T @ G], axis=0)
        if need_dx:
            dX = P.T @ (G @ W[d_in:].T)
            dX[: block.n_dst] += G @ W[:d_in].T
    else:
        dW = A.T @ G
        if need_dx:
            dX = P.T @ (G @ W.T)
    return dW, db, dX


def sgd_update(params: List[np.ndarray], grads: List[np.ndarray], lr: float):
    """Plain gradient descent: p <- p - lr * g."""
    return [np.asarray(p, np.float64) - lr * np.asarray(g, np.float64) for p, g in zip(params, grads)]


def forward_all(blocks: Sequence[Block], X: np.ndarray, weights, kind="sage", aggr="mean"):
    """Layers 1..L; layer i uses block b_{L-i} (SURVEY §8 notation)."""
    L = len(blocks)
    Hs = [np.asarray(X, dtype=np.float64)]
    As = []
    for i in range(1, L + 1):
        blk = blocks[L - i]
        W, b = weights[i - 1]
        Hout, A = layer_fwd(blk, Hs[-1], W, b, relu=(i < L), kind=kind, aggr=aggr)
        Hs.append(Hout)
        As.append(A)
    return Hs, As


def train_step(indptr, indices, feats, d, labels, seeds, fanouts, rng_seed, weights,
               lr: float, n_global: Optional[int] = None, kind="sage", aggr="mean") -> Dict:
    """One iteration of Algorithm 1 on one rank's seed slice:
    sample -> gather -> L x (Aggregate, Combine) -> loss -> backward -> SGD.

    Gradients are NOT all-reduced here; the caller sums them over ranks."""
    from .gather import gather_rows

    seeds = np.asarray(seeds, dtype=np.int64)
    n_global = int(n_global or seeds.size)
    frontiers, blocks = sample_blocks(indptr, indices, seeds, fanouts, rng_seed)
    X = gather_rows(feats, frontiers[-1])[:, :d]
    Hs, As = forward_all(blocks, X, weights, kind, aggr)
    L = len(blocks)
    loss, G = ce_loss(Hs[-1], np.asarray(labels)[seeds], n_global)
    grads = [None] * L
    for i in range(L, 0, -1):
        blk = blocks[L - i]
        W, _ = weights[i - 1]
        dW, db, dX = layer_bwd(blk, Hs[i - 1], As[i - 1], Hs[i], W, G, relu=(i < L),
                               need_dx=(i > 1), kind=kind, aggr=aggr)
        grads[i - 1] = (dW, db)
        G = dX
    new_w = [tuple(sgd_update([W, b], [dW, db], lr)) for (W, b), (dW, db) in zip(weights, grads)]
    return dict(frontiers=frontiers, blocks=blocks, X=X, Hs=Hs, As=As, loss=loss,
                grads=grads, new_weights=new_w)


def flop_count(n_rows: Sequence[int], nnz: Sequence[int], dims: Sequence[int]) -> int:
    """sum_l 2 |V_l| d_{l-1} d_l (combine) + sum_l |E_l| d_{l-1} (aggregate)."""
    f = 0
    for l in range(1, len(dims)):
        f += 2 * int(n_rows[l - 1]) * int(dims[l - 1]) * int(dims[l])
        f += int(nnz[l - 1]) * int(dims[l - 1])
    return f
