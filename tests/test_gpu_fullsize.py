"""-m gpu parity at BASELINE.json's full sizes, in the launch configuration
bench.py times (Trainer, Eq.4 prefetch of device seeds on its own stream,
step on a high-priority stream), against the oracle on the same seeded
inputs, for configs[0..3] -- Cora (ratio 0.2, d = 1433), arxiv (3 layers,
ratio 0.5), Reddit (fanout 25, d = 602, ratio 0.1 and 1.0: misses read
zero-copy from pinned host memory / the whole table in HBM), products (the
bench workload) -- each in tf32 (the bench's GEMMs) and fp32 (parity mode);
configs[4] (papers100M) is tests/test_gpu_papers100m.py.

Per case, the whole step (full_step_check): sampling, relabelling, gather
and hit counters bit-exact over EVERY row; each layer elementwise on the
GPU's own input (a large layer on 2048 sampled dst rows as a row-restricted
block -- rows are independent problems); loss; every weight/bias gradient
elementwise against the oracle's backward chain run on the GPU's forward
values (condition-aware, one rtol per GEMM stage from the loss); every
gradient's direction vs the oracle's own fp64 step.
"""
import numpy as np
import pytest
import torch

import oracle
from oracle.cache import access_counts, cache_slots
from oracle.layers import agg_matrix, ce_loss, layer_bwd, layer_fwd, train_step
from oracle.sampler import Block, sample_blocks
from paper_2404_09544_b200 import gnnv
from synth import BASE_RNG_SEED, CONFIGS, epoch_seeds, init_weights
from synth.store import shared_graph

from gpu_util import (_blk, assert_close_cond, bf16_round, blocks_to_host, check_backward_chain, check_forward_chain, lib,
                      normwise, read_bf16, read_f32, read_i32, sub_block)

pytestmark = pytest.mark.gpu

RTOL = {0: 1e-5, 2: 4e-3}  # fp32 / tf32, as test_gpu_parity (reading Q17, Q22)


def pipelined_step(tr, d_seeds, n, n_global, rng_seed, lr):
    """One step as bench.py runs it: the batch is prefetched (sample +
    gather on the trainer's side stream) with device seeds ordered on their
    own stream, then consumed by the step on a high-priority stream."""
    pf = torch.cuda.Stream()
    main = torch.cuda.Stream(priority=-1)
    torch.cuda.synchronize()
    tr.prefetch(d_seeds.data_ptr(), n, rng_seed, on_host=False, stream=pf)
    tr.step(d_seeds.data_ptr(), n, n_global, rng_seed, lr, on_host=False, want_loss=False, stream=main)
    loss = tr.read_loss(stream=main)
    torch.cuda.synchronize()
    return loss


def check_blocks_and_gather(gd, tr, ref_frontiers, ref_blocks, ratio):
    hb = blocks_to_host(tr.blocks)
    assert len(hb) == len(ref_blocks)
    for h, ((nd, ns, ptr, idx, F), ob) in enumerate(zip(hb, ref_blocks)):
        assert (nd, ns) == (ob.n_dst, ob.n_src), (h, nd, ns, ob.n_dst, ob.n_src)
        np.testing.assert_array_equal(F, ref_frontiers[h + 1], err_msg=f"F_{h + 1}")
        np.testing.assert_array_equal(ptr, ob.indptr, err_msg=f"indptr hop {h}")
        np.testing.assert_array_equal(idx, ob.indices, err_msg=f"indices hop {h}")
    FL = ref_frontiers[-1]
    slot, owner, _ = cache_slots(gd.indptr, ratio)
    # X holds F_L; or only the dst prefix F_{L-1} when the whole table is
    # cached (the layer-1 aggregation then reads the cache table directly);
    # or nothing (-1) when the tf32 layer-1 GEMMs gather H_dst from the table
    # too.  With the whole table, the rows layer 1 reads are table rows
    # rowidx[u]: rowidx must be the oracle's slot of every F_L row and those
    # table rows the feature rows, bit for bit.
    lvl = tr.x_level()
    L = len(ref_blocks)
    assert lvl in ((L - 1, -1) if ratio == 1.0 else (L,))
    if lvl >= 0:
        Fx = ref_frontiers[lvl]
        p0, s0 = tr.activation(0)
        X = read_f32(p0, len(Fx), s0)
        assert X.tobytes() == oracle.gather_rows(gd.feats, Fx).tobytes(), "gathered rows"
    if tr.dw16():  # layer 1's bf16 operand copy of X's dst prefix: the rounded feature rows + the ones column
        Fx = ref_frontiers[L - 1]
        px, _, ld = tr.dw16_operands()
        X16 = read_bf16(px, len(Fx), ld)
        Xr = oracle.gather_rows(gd.feats, Fx)[:, : gd.d]
        np.testing.assert_array_equal(X16[:, : gd.d], bf16_round(Xr), err_msg="bf16 copy of the gathered rows")
        np.testing.assert_array_equal(X16[:, gd.d], 1.0)
    # a trainer that leaves its last hop unrelabelled (gnnv_trainer_last_rows)
    # resolves and counts the rows of F_{L-1}: the last hop's edges carry
    # their table rows themselves (checked through blocks_to_host above)
    if tr.last_rows():
        FL = ref_frontiers[-2]
    if ratio == 1.0:
        pr, pt = tr.rowidx()
        ridx = read_i32(pr, len(FL))
        np.testing.assert_array_equal(ridx, slot[FL], err_msg="cache rows of F_L")
        pick = np.random.default_rng(1).choice(len(FL), min(len(FL), 4096), replace=False)
        for u in pick[:64]:  # the table rows themselves (cache build), a sample
            row = read_f32(pt + int(ridx[u]) * gd.stride * 4, 1, gd.stride)
            assert row.tobytes() == oracle.gather_rows(gd.feats, FL[u:u + 1]).tobytes(), ("table row", u)
    cnt = access_counts(slot, owner, FL)
    assert tr.stats().tolist() == [cnt["rows"], cnt["hits_local"], cnt["hits_peer"], cnt["misses_host"]]
    return hb


_GRAPHS = {}
_REFS = {}


def graph_of(name):
    """(GraphData, gnnv.Graph) of a config, generated once per session
    (through the box's shared host store, synth.store)."""
    if name not in _GRAPHS:
        lib()
        gd = shared_graph(name)
        _GRAPHS[name] = (gd, gnnv.Graph.from_data(gd))
    return _GRAPHS[name]


def dims_of(name, gd):
    cfg = CONFIGS[name]
    return [gd.d] + [cfg["hidden"]] * (len(cfg["fanouts"]) - 1) + [gd.C]


T_BENCH = 10  # a bench-timed iteration index (after the warm-up)


def oracle_ref(name):
    """The oracle's own fp64 step on iteration T_BENCH's batch (independent of
    the cache ratio and the GEMM precision, so computed once per config)."""
    if name not in _REFS:
        gd, _ = graph_of(name)
        cfg = CONFIGS[name]
        B = cfg["batch"]
        seeds = epoch_seeds(gd.n, 0)[T_BENCH * B:(T_BENCH + 1) * B]
        w = init_weights(dims_of(name, gd))
        ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, cfg["fanouts"],
                         BASE_RNG_SEED + T_BENCH, w, 0.01)
        _REFS[name] = (seeds, w, ref)
    return _REFS[name]


def full_step_check(name, ratio, prec, max_rows=2048):
    """One step of config `name` as bench.py runs it (Trainer, Eq.4 prefetch
    of device seeds, step on a high-priority stream) against the oracle:
    blocks, frontiers, gathered rows and counters bit-exact over every row;
    every layer of the forward chain elementwise on the GPU's own input (at
    most max_rows sampled dst rows of a large layer, as row-restricted
    blocks); the loss; every dW/db elementwise through the oracle's backward
    chain on the GPU's forward values (condition-aware, one rtol per GEMM
    stage from the loss); every gradient's direction vs the oracle's own
    fp64 step."""
    gd, g = graph_of(name)
    cfg = CONFIGS[name]
    dims = dims_of(name, gd)
    L = len(cfg["fanouts"])
    seeds, w, ref = oracle_ref(name)
    B = cfg["batch"]
    cache = gnnv.Cache(g, ratio)
    tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, w, prec=prec)
    try:
        d_seeds = torch.as_tensor(seeds.astype(np.int32)).cuda()
        loss = pipelined_step(tr, d_seeds, B, B, BASE_RNG_SEED + T_BENCH, 0.01)
        hb = check_blocks_and_gather(gd, tr, ref["frontiers"], ref["blocks"], ratio)
        grads = gnnv.unflat_params(tr.grads(), dims)
        rtol = RTOL[prec]
        assert abs(loss - ref["loss"]) <= (1e-4 if prec == 0 else 5e-3) * abs(ref["loss"]), (loss, ref["loss"])
        X0 = oracle.gather_rows(gd.feats, hb[L - 1][4])[:, : dims[0]] if tr.x_level() < L else None
        H, Aagg, blks = check_forward_chain(tr, hb, dims, w, rtol, name, X0=X0, max_rows=max_rows)
        check_backward_chain(tr, blks, H, Aagg, dims, w, grads, gd.labels[seeds], B, rtol, name)
        # and the direction of every gradient vs the oracle's own fp64 step
        for i, ((gW, gb), (rW_, rb_)) in enumerate(zip(grads, ref["grads"])):
            for a_, b_ in ((gW, rW_), (gb, rb_)):
                cos = float(np.dot(a_.ravel(), b_.ravel()) / (np.linalg.norm(a_) * np.linalg.norm(b_) + 1e-30))
                assert cos > 0.98, (name, i, cos)
    finally:
        tr.free()
        cache.free()


# BASELINE.json configs[0..3] at their own cache ratios (and the full-cache
# end of configs[2]'s sweep); tf32 = the bench's precision, fp32 = parity mode
CASES = [("cora", 0.2), ("arxiv", 0.5), ("reddit", 0.1), ("reddit", 1.0), ("products", 1.0)]


@pytest.mark.parametrize("prec", [2, 0], ids=["tf32", "fp32"])
@pytest.mark.parametrize("name,ratio", CASES, ids=[f"{n}@{r}" for n, r in CASES])
def test_full_step(name, ratio, prec):
    full_step_check(name, ratio, prec)
