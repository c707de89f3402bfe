"""Pins for oracle/layers.py: brute-force dense adjacency, SPEC examples
(S:325), torch float64 autograd, central finite differences,
permutation invariance, loss decrease."""
import numpy as np
import pytest
import torch

from oracle.layers import (agg_matrix, ce_loss, flop_count, forward_all, layer_bwd,
                           layer_fwd, train_step)
from oracle.sampler import Block, sample_blocks
from synth import chung_lu_graph, init_weights, make_features, make_labels, tiny_graph


def _random_block(rng, n_dst=7, extra=9, maxdeg=4):
    n_src = n_dst + extra
    counts = rng.integers(0, maxdeg + 1, size=n_dst)
    idx = []
    for c in counts:
        idx += rng.choice(n_src, size=int(c), replace=False).tolist()
    indptr = np.concatenate([[0], np.cumsum(counts)])
    return Block(n_dst=n_dst, n_src=n_src, indptr=indptr, indices=np.array(idx, dtype=np.int64),
                 src_global=np.arange(n_src))


@pytest.mark.parametrize("kind,aggr", [("sage", "mean"), ("sage", "sum"), ("gcn", "mean"), ("gcn", "sum")])
def test_aggregation_brute_force_dense(kind, aggr):
    rng = np.random.default_rng(1)
    b = _random_block(rng)
    H = rng.standard_normal((b.n_src, 5))
    D = np.zeros((b.n_dst, b.n_src))
    for v in range(b.n_dst):
        nb = b.indices[b.indptr[v]:b.indptr[v + 1]]
        c = len(nb)
        for u in nb:
            D[v, u] += 1.0
        if kind == "gcn":
            D[v, v] += 1.0
        if aggr == "mean":
            denom = c + (1 if kind == "gcn" else 0)
            if denom:
                D[v] /= denom
    P = agg_matrix(b, kind, aggr)
    np.testing.assert_allclose(P.toarray(), D, rtol=0, atol=1e-15)
    np.testing.assert_allclose(P @ H, D @ H, rtol=1e-13, atol=1e-13)


def test_isolated_vertex_identity():
    """isolated vertex, mean aggregate, identity weights -> output = input.
    SAGE reading: W_s = I, b = 0; a zero-neighbour row aggregates to 0 (Q15)."""
    g = tiny_graph("isolated", d=4)
    F, blocks = sample_blocks(g.indptr, g.indices, [5], [3], 0)
    d = 4
    W = np.concatenate([np.eye(d), np.zeros((d, d))])
    H, A = layer_fwd(blocks[0], g.feats[F[1], :d], W, np.zeros(d), relu=False)
    np.testing.assert_array_equal(H, g.feats[[5], :d].astype(np.float64))
    assert (A == 0).all()
    Hg, _ = layer_fwd(blocks[0], g.feats[F[1], :d], np.eye(d), np.zeros(d), relu=False, kind="gcn")
    np.testing.assert_array_equal(Hg, g.feats[[5], :d].astype(np.float64))


def test_flop_count_example():
    assert flop_count([3], [0], [2, 2]) == 24
    assert flop_count([0], [0], [5, 7]) == 0


def _torch_forward(blocks, X, weights, labels, n_global, kind, aggr):
    L = len(blocks)
    H = torch.tensor(X, dtype=torch.float64)
    params = []
    for i in range(1, L + 1):
        b = blocks[L - i]
        W = torch.tensor(weights[i - 1][0], dtype=torch.float64, requires_grad=True)
        bb = torch.tensor(weights[i - 1][1], dtype=torch.float64, requires_grad=True)
        params += [W, bb]
        rows = torch.repeat_interleave(torch.arange(b.n_dst), torch.tensor(np.diff(b.indptr)))
        cols = torch.tensor(b.indices)
        S = torch.zeros(b.n_dst, H.shape[1], dtype=torch.float64).index_add(0, rows, H[cols])
        c = torch.tensor(np.diff(b.indptr), dtype=torch.float64)[:, None]
        d_in = H.shape[1]
        if kind == "sage":
            A = S / c.clamp(min=1) if aggr == "mean" else S
            Z = H[: b.n_dst] @ W[:d_in] + A @ W[d_in:] + bb
        else:
            A = (H[: b.n_dst] + S) / (c + 1) if aggr == "mean" else H[: b.n_dst] + S
            Z = A @ W + bb
        H = torch.relu(Z) if i < L else Z
    y = torch.tensor(np.asarray(labels, dtype=np.int64))
    loss = torch.nn.functional.cross_entropy(H, y, reduction="sum") / n_global
    loss.backward()
    return float(loss), [(p.grad.numpy()) for p in params]


@pytest.mark.parametrize("kind,aggr", [("sage", "mean"), ("sage", "sum"), ("gcn", "mean")])
def test_step_grads_match_torch_autograd(kind, aggr):
    indptr, indices = chung_lu_graph(600, 4000, 0.5, seed=3)
    d, C = 6, 5
    feats = make_features(600, d)
    labels = make_labels(600, C)
    seeds = np.random.default_rng(4).permutation(600)[:16]
    dims = [d, 8, 7, C]
    w = init_weights(dims, kind=kind)
    out = train_step(indptr, indices, feats, d, labels, seeds, [4, 3, 2], 55, w, lr=0.1,
                     n_global=40, kind=kind, aggr=aggr)
    tl, tg = _torch_forward(out["blocks"], out["X"], w, labels[seeds], 40, kind, aggr)
    assert abs(tl - out["loss"]) < 1e-12
    for i, (dW, db) in enumerate(out["grads"]):
        np.testing.assert_allclose(dW, tg[2 * i], rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(db, tg[2 * i + 1], rtol=1e-10, atol=1e-13)


def test_central_finite_differences():
    """gradient vs central differences <= 1e-4 relative."""
    indptr, indices = chung_lu_graph(60, 300, 0.5, seed=8)
    d, C = 3, 3
    feats = make_features(60, d)
    labels = make_labels(60, C)
    seeds = [1, 5, 9, 22]
    w = [(W.astype(np.float64), b.astype(np.float64)) for W, b in init_weights([d, 4, C])]
    base = train_step(indptr, indices, feats, d, labels, seeds, [3, 2], 7, w, lr=0.0)

    def loss_of(ww):
        Hs, _ = forward_all(base["blocks"], base["X"], ww)
        return ce_loss(Hs[-1], labels[seeds], len(seeds))[0]

    eps = 1e-6
    for li in range(2):
        for which in range(2):
            P = w[li][which]
            G = base["grads"][li][which]
            it = np.nditer(P, flags=["multi_index"])
            for _ in it:
                ix = it.multi_index
                wp = [(W.copy(), b.copy()) for W, b in w]
                wm = [(W.copy(), b.copy()) for W, b in w]
                wp[li][which][ix] += eps
                wm[li][which][ix] -= eps
                fd = (loss_of(wp) - loss_of(wm)) / (2 * eps)
                assert abs(fd - G[ix]) <= 1e-4 * max(abs(fd), abs(G[ix]), 1e-3)


def test_permutation_invariance():
    """relabelling src-only vertices leaves the dst outputs unchanged."""
    rng = np.random.default_rng(6)
    b = _random_block(rng, n_dst=5, extra=11)
    H = rng.standard_normal((b.n_src, 4))
    W = rng.standard_normal((8, 3))
    bias = rng.standard_normal(3)
    out, _ = layer_fwd(b, H, W, bias, relu=True)
    perm = np.concatenate([np.arange(b.n_dst), b.n_dst + rng.permutation(b.n_src - b.n_dst)])
    inv = np.argsort(perm)
    b2 = Block(b.n_dst, b.n_src, b.indptr, inv[b.indices], b.src_global[perm])
    out2, _ = layer_fwd(b2, H[perm], W, bias, relu=True)
    np.testing.assert_allclose(out, out2, rtol=1e-12, atol=1e-12)


def test_loss_non_increasing_small_instance():
    """loss non-increasing over the first 10 steps at lr 1e-2 (fixed batch)."""
    indptr, indices = chung_lu_graph(300, 2400, 0.5, seed=12)
    d, C = 8, 4
    feats = make_features(300, d)
    labels = make_labels(300, C)
    seeds = np.arange(32)
    w = [(W.astype(np.float64), b.astype(np.float64)) for W, b in init_weights([d, 16, C])]
    prev = np.inf
    for _ in range(10):
        out = train_step(indptr, indices, feats, d, labels, seeds, [5, 5], 3, w, lr=1e-2)
        assert out["loss"] <= prev + 1e-12
        prev = out["loss"]
        w = out["new_weights"]


def test_rank_split_gradients_sum_to_concatenated():
    """sum over ranks of the 1/B_global-scaled gradients equals
    the gradient of the concatenated batch."""
    indptr, indices = chung_lu_graph(2000, 16000, 0.5, seed=1)
    d, C = 5, 4
    feats = make_features(2000, d)
    labels = make_labels(2000, C)
    seeds = np.random.default_rng(2).permutation(2000)[:40]
    w = init_weights([d, 6, C])
    full = train_step(indptr, indices, feats, d, labels, seeds, [4, 3], 9, w, lr=0.0)
    parts = [train_step(indptr, indices, feats, d, labels, s, [4, 3], 9, w, lr=0.0, n_global=40)
             for s in (seeds[:17], seeds[17:])]
    assert abs(sum(p["loss"] for p in parts) - full["loss"]) < 1e-12
    for li in range(2):
        for j in range(2):
            np.testing.assert_allclose(parts[0]["grads"][li][j] + parts[1]["grads"][li][j],
                                       full["grads"][li][j], rtol=1e-10, atol=1e-13)
