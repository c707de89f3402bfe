"""-m gpu: parity on the papers100M-shaped graph, BASELINE.json configs[4]
(111M nodes, 1.6B CSR entries, 128-d, fanouts [15,10,5], batch 8192).
Generating the graph takes minutes and ~65 GB of host memory (kept in the
box's shared store, synth.store, for the bench); GNNV_SKIP_PAPERS100M=1
skips it on a box without that memory.

One rank's batch, in the bench launch configuration (Trainer, Eq.4
prefetch, tf32): blocks, frontiers, every gathered row (the cache-table row
of every F_L row) and the hit counters bit-exact against the oracle; layer 1
(aggregation over the sampled table rows + the tf32 GEMMs) elementwise on
2048 sampled dst rows against the oracle's layer on the same rows; the loss
finite.  The cache is the full table replicated on the one GPU of the box
(the 8-GPU sharded placement is exercised by tests/test_gpu_sharded.py).
"""
import os

import numpy as np
import pytest
import torch

import oracle
from oracle.cache import access_counts, cache_slots
from oracle.sampler import sample_blocks
from paper_2404_09544_b200 import gnnv
from oracle.layers import layer_fwd
from oracle.sampler import Block
from synth import BASE_RNG_SEED, CONFIGS, epoch_seeds, init_weights
from synth.store import shared_graph

from gpu_util import assert_close_cond, blocks_to_host, lib, read_bf16, read_f32, read_i32

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(os.environ.get("GNNV_SKIP_PAPERS100M") == "1", reason="GNNV_SKIP_PAPERS100M=1"),
]


def test_papers100m_batch_bit_exact():
    lib()
    cfg = CONFIGS["papers100m"]
    gd = shared_graph("papers100m")
    g = gnnv.Graph.from_data(gd)
    cache = gnnv.Cache(g, cfg["ratio"])
    dims = [gd.d] + [cfg["hidden"]] * (len(cfg["fanouts"]) - 1) + [gd.C]
    B = cfg["batch"]
    w = init_weights(dims)
    tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, w, prec=gnnv.PREC_TF32)
    seeds = epoch_seeds(gd.n, 0)[:B]
    rs = BASE_RNG_SEED + 1
    d_seeds = torch.as_tensor(seeds.astype(np.int32)).cuda()
    pf, main = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    torch.cuda.synchronize()
    tr.prefetch(d_seeds.data_ptr(), B, rs, on_host=False, stream=pf)
    tr.step(d_seeds.data_ptr(), B, B, rs, 0.01, on_host=False, want_loss=False, stream=main)
    loss = tr.read_loss(stream=main)
    assert np.isfinite(loss)
    F, blocks = sample_blocks(gd.indptr, gd.indices, seeds, cfg["fanouts"], rs)
    hb = blocks_to_host(tr.blocks)
    for h, ((nd, ns, ptr, idx, Fg), ob) in enumerate(zip(hb, blocks)):
        assert (nd, ns) == (ob.n_dst, ob.n_src)
        np.testing.assert_array_equal(Fg, F[h + 1])
        np.testing.assert_array_equal(ptr, ob.indptr)
        np.testing.assert_array_equal(idx, ob.indices)
    FL = F[-1]
    slot, owner, _ = cache_slots(gd.indptr, cfg["ratio"])
    lvl = tr.x_level()  # whole table cached: X holds the dst prefix F_{L-1}, or nothing (-1)
    if lvl >= 0:
        Fx = F[lvl]
        p0, s0 = tr.activation(0)
        X = read_f32(p0, len(Fx), s0)
        assert X.tobytes() == oracle.gather_rows(gd.feats, Fx).tobytes()
    if tr.last_rows():  # the last hop unrelabelled: rowidx and the counters cover F_{L-1}
        FL = F[-2]
    pr, pt = tr.rowidx()  # the rows layer 1 reads: table rows rowidx[u] = slot of F_L[u]
    np.testing.assert_array_equal(read_i32(pr, len(FL)), slot[FL])
    cnt = access_counts(slot, owner, FL)
    assert tr.stats().tolist() == [cnt["rows"], cnt["hits_local"], cnt["hits_peer"], cnt["misses_host"]]
    # layer 1 on 2048 sampled dst rows of F_{L-1}: its input rows are the
    # feature rows of the sampled neighbours (read by the GPU from the table)
    L = len(cfg["fanouts"])
    nd, ns, ptr, idx, Fg = hb[L - 1]
    # the fp32 H^1 holds layer 2's dst prefix only (bf16 intermediates, reading Q30)
    n_keep = hb[L - 2][0] if (tr.l2push() or tr.bf16act()) else nd
    rows = np.sort(np.random.default_rng(0).choice(n_keep, 2048, replace=False))
    cnt = np.diff(ptr)[rows]
    nbr = np.concatenate([idx[ptr[r]:ptr[r + 1]] for r in rows])
    blk = Block(n_dst=len(rows), n_src=len(rows) + nbr.size, indptr=np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64),
                indices=(len(rows) + np.arange(nbr.size)).astype(np.int64), src_global=None)
    Hs = oracle.gather_rows(gd.feats, np.concatenate([Fg[rows], Fg[nbr]]))[:, : gd.d]
    W1, b1 = w[0]
    Ho, _ = layer_fwd(blk, Hs, W1, b1, True)
    Hm, _ = layer_fwd(blk, Hs, W1, b1, True, absval=True)
    p1, s1 = tr.activation(1)
    H1 = read_f32(p1, n_keep, s1)[rows, : dims[1]]
    assert_close_cond(H1, Ho, Hm, 4e-3, "papers100m layer 1 (sampled rows)")
    if tr.bf16act():  # the bf16 copy of H^1 (every row): layer 1 plus bf16 rounding, on rows beyond the prefix too
        rows = np.sort(np.random.default_rng(1).choice(nd, 2048, replace=False))
        cnt = np.diff(ptr)[rows]
        nbr = np.concatenate([idx[ptr[r]:ptr[r + 1]] for r in rows])
        blk = Block(n_dst=len(rows), n_src=len(rows) + nbr.size,
                    indptr=np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64),
                    indices=(len(rows) + np.arange(nbr.size)).astype(np.int64), src_global=None)
        Hs = oracle.gather_rows(gd.feats, np.concatenate([Fg[rows], Fg[nbr]]))[:, : gd.d]
        Ho, _ = layer_fwd(blk, Hs, W1, b1, True)
        Hm, _ = layer_fwd(blk, Hs, W1, b1, True, absval=True)
        p16, ld16 = tr.activation16(1)
        H16 = read_bf16(p16, nd, ld16)[rows, : dims[1]]
        assert_close_cond(H16, Ho, (4e-3 + 2.0 ** -8) / 4e-3 * Hm, 4e-3, "papers100m bf16 copy of layer 1")
    print(f"papers100m: frontiers {[len(f) for f in F]}, edges {[b.nnz for b in blocks]}, loss {loss:.5f}")
