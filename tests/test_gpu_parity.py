"""-m gpu parity tests: the CUDA path (through the C-ABI) vs the CPU oracle on
the same seeded inputs.  Integer work (sampling, relabelling, cache slots,
hit counters) and gathered rows are bit-exact; floating point within the
condition-aware tolerance of reading Q17 (1e-5 fp32, 2e-2 bf16)."""
import os

import numpy as np
import pytest
import torch

import oracle
from oracle.cache import access_counts, cache_slots
from oracle.layers import agg_matrix, ce_loss, layer_bwd, layer_fwd, train_step
from oracle.sampler import Block, sample_blocks
from paper_2404_09544_b200 import gnnv
from synth import CONFIGS, epoch_seeds, init_weights, make_graph, row_stride, tiny_graph

from gpu_util import check_backward_chain, check_forward_chain, sub_block, assert_close_cond, blocks_to_host, dev_f32, dev_i32, bf16_round, layer1_aggregate, lib, normwise, read_activation, read_bf16, read_f32, read_i32

pytestmark = pytest.mark.gpu

RTOL32 = 1e-5
RTOL16 = 2e-2
# tf32: two operands truncated to a 10-bit mantissa (<= 2^-10 each) -> 2e-3 of
# the |A||B| magnitude, plus fp32 accumulation; 4e-3 keeps a 2x margin.
RTOL_TF32 = 4e-3
RTOL = {0: RTOL32, 1: RTOL16, 2: RTOL_TF32}


@pytest.fixture(scope="module")
def mini():
    lib()
    gd = make_graph("mini")
    g = gnnv.Graph.from_data(gd)
    return gd, g


@pytest.fixture
def option():
    """gnnv.set_option(name, value) for one test; back to the environment after."""
    names = []

    def set_(name, value):
        gnnv.set_option(name, value)
        names.append(name)

    yield set_
    for n in names:
        gnnv.set_option(n, -1)


@pytest.fixture(scope="module")
def cora():
    lib()
    gd = make_graph("cora")
    g = gnnv.Graph.from_data(gd)
    return gd, g


def gpu_sample(g, seeds, fanouts, rng_seed, max_seeds=None):
    blocks = gnnv.Blocks(g, max_seeds or len(seeds), fanouts)
    ds = dev_i32(seeds)
    blocks.sample(ds, len(seeds), rng_seed)
    return blocks, blocks_to_host(blocks)


def assert_blocks_equal(host_blocks, oF, oB):
    assert len(host_blocks) == len(oB)
    for h, ((nd, ns, ptr, idx, F), ob) in enumerate(zip(host_blocks, oB)):
        assert nd == ob.n_dst and ns == ob.n_src, (h, nd, ns, ob.n_dst, ob.n_src)
        np.testing.assert_array_equal(F, oF[h + 1], err_msg=f"frontier F_{h + 1}")
        np.testing.assert_array_equal(ptr, ob.indptr, err_msg=f"indptr hop {h}")
        np.testing.assert_array_equal(idx, ob.indices, err_msg=f"indices hop {h}")


# ------------------------------------------------------------- sampling
@pytest.mark.parametrize("rng_seed", [0, 1, 0x5EED, 2**63 + 12345])
@pytest.mark.parametrize("n_seeds", [1, 300, 512])
def test_sample_bit_exact_mini(mini, rng_seed, n_seeds):
    gd, g = mini
    seeds = epoch_seeds(gd.n, 0)[:n_seeds]
    fan = CONFIGS["mini"]["fanouts"]
    _, hb = gpu_sample(g, seeds, fan, rng_seed, max_seeds=512)
    oF, oB = sample_blocks(gd.indptr, gd.indices, seeds, fan, rng_seed)
    assert_blocks_equal(hb, oF, oB)


@pytest.mark.parametrize("fan", [[1], [3, 2], [25, 10], [32, 32, 4], [5, 5, 5, 5]])
def test_sample_bit_exact_fanouts(mini, fan):
    gd, g = mini
    seeds = epoch_seeds(gd.n, 1)[:97]
    _, hb = gpu_sample(g, seeds, fan, 77)
    oF, oB = sample_blocks(gd.indptr, gd.indices, seeds, fan, 77)
    assert_blocks_equal(hb, oF, oB)


def test_sample_bit_exact_cora(cora):
    gd, g = cora
    cfg = CONFIGS["cora"]
    for t in range(3):
        seeds = epoch_seeds(gd.n, 0)[t * cfg["batch"]:(t + 1) * cfg["batch"]]
        _, hb = gpu_sample(g, seeds, cfg["fanouts"], 0x5EED + t)
        oF, oB = sample_blocks(gd.indptr, gd.indices, seeds, cfg["fanouts"], 0x5EED + t)
        assert_blocks_equal(hb, oF, oB)


@pytest.mark.parametrize("kind", ["path5", "star10", "isolated", "twostar", "clique"])
def test_sample_tiny_graphs(kind):
    lib()
    gd = tiny_graph(kind)
    g = gnnv.Graph.from_data(gd)
    seeds = list(range(min(gd.n, 3)))
    for fan in ([2], [3, 3], [10, 1]):
        _, hb = gpu_sample(g, seeds, fan, 5)
        oF, oB = sample_blocks(gd.indptr, gd.indices, seeds, fan, 5)
        assert_blocks_equal(hb, oF, oB)


def test_sample_repeat_calls_and_reset(mini):
    """A blocks handle is reusable: tags are reset after every call."""
    gd, g = mini
    fan = [15, 10, 5]
    blocks = gnnv.Blocks(g, 512, fan)
    perm = epoch_seeds(gd.n, 2)
    for t in range(4):
        seeds = perm[t * 200:(t + 1) * 200 + t]
        blocks.sample(dev_i32(seeds), len(seeds), 1000 + t)
        hb = blocks_to_host(blocks)
        oF, oB = sample_blocks(gd.indptr, gd.indices, seeds, fan, 1000 + t)
        assert_blocks_equal(hb, oF, oB)


def test_sample_errors(mini):
    gd, g = mini
    blocks = gnnv.Blocks(g, 8, [3])
    blocks.sample(dev_i32([1, 2, 2]), 3, 0)
    with pytest.raises(gnnv.GnnvError) as e:
        blocks.info(sync=True)
    assert e.value.status == gnnv.ERR_PARAM
    blocks.sample(dev_i32([1, gd.n + 5]), 2, 0)
    with pytest.raises(gnnv.GnnvError):
        blocks.info(sync=True)
    # the handle recovers after an error
    blocks.sample(dev_i32([1, 2, 3]), 3, 0)
    hb = blocks_to_host(blocks)
    oF, oB = sample_blocks(gd.indptr, gd.indices, [1, 2, 3], [3], 0)
    assert_blocks_equal(hb, oF, oB)
    with pytest.raises(gnnv.GnnvError):
        blocks.sample(dev_i32([1]), 9, 0)  # n_seeds > max_seeds
    with pytest.raises(gnnv.GnnvError):
        gnnv.Blocks(g, 8, [0])  # fanout < 1


# ----------------------------------------------------------- cache + gather
@pytest.mark.parametrize("ratio,policy", [(0.0, 1), (0.2, 1), (0.5, 1), (1.0, 1), (0.7, 0)])
def test_cache_slots_bit_exact(mini, ratio, policy):
    gd, g = mini
    c = gnnv.Cache(g, ratio, policy=policy)
    v = c.info()
    slot, _, _ = cache_slots(gd.indptr, ratio, policy)
    from gpu_util import read_i32
    np.testing.assert_array_equal(read_i32(v.d_slot, gd.n), slot)
    assert v.capacity == int((slot >= 0).sum())


@pytest.mark.parametrize("ratio,placement,G", [(0.3, 0, 1), (0.0, 0, 1), (1.0, 0, 1), (0.45, 2, 4), (1.0, 2, 3)])
def test_gather_bit_exact(mini, ratio, placement, G):
    gd, g = mini
    c = gnnv.Cache(g, ratio, placement=placement, virtual_shards=G)
    fan = CONFIGS["mini"]["fanouts"]
    seeds = epoch_seeds(gd.n, 0)[:512]
    blocks, hb = gpu_sample(g, seeds, fan, 3)
    FL = hb[-1][4]
    X = torch.empty((blocks.info(sync=False)[-1].max_src, gd.stride), dtype=torch.float32, device="cuda")
    stats = torch.zeros(4, dtype=torch.int64, device="cuda")
    gnnv.gather(c, blocks, X, stats)
    torch.cuda.synchronize()
    got = X[: len(FL)].cpu().numpy()
    ref = oracle.gather_rows(gd.feats, FL)
    assert got.tobytes() == ref.tobytes()
    slot, owner, _ = cache_slots(gd.indptr, ratio, world=G)
    cnt = access_counts(slot, owner, FL, me=0)
    s = stats.cpu().numpy()
    assert s.tolist() == [cnt["rows"], cnt["hits_local"], cnt["hits_peer"], cnt["misses_host"]]


# ------------------------------------------------------------------ layers
def padded(arr, cap):
    """Device copy of `arr` in a buffer of `cap` rows (capacity-sized, as the
    layer API requires); the rows beyond are NaN and must never matter."""
    t = torch.full((int(cap), arr.shape[1]), float("nan"), device="cuda")
    t[: arr.shape[0]] = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float32)).cuda()
    return t


def _oracle_block(hb, h):
    nd, ns, ptr, idx, F = hb[h]
    return Block(n_dst=nd, n_src=ns, indptr=ptr.astype(np.int64), indices=idx.astype(np.int64), src_global=F)


@pytest.mark.parametrize("kind,aggr", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("prec", [0, 1, 2])
def test_layer_fwd_bwd_parity(mini, kind, aggr, prec):
    gd, g = mini
    fan = CONFIGS["mini"]["fanouts"]
    seeds = epoch_seeds(gd.n, 0)[:300]
    blocks, hb = gpu_sample(g, seeds, fan, 11, max_seeds=512)
    L = len(fan)
    rng = np.random.default_rng(0)
    kname = "sage" if kind == 0 else "gcn"
    aname = "mean" if aggr == 0 else "sum"
    rtol = RTOL[prec]
    for layer, (d_in, d_out) in zip(range(1, L + 1), [(gd.d, 64), (64, 64), (64, gd.C)]):
        h = L - layer
        ob = _oracle_block(hb, h)
        s_in = gd.stride if layer == 1 else row_stride(d_in)
        Hsrc = np.zeros((ob.n_src, s_in), np.float32)
        Hsrc[:, :d_in] = rng.standard_normal((ob.n_src, d_in)).astype(np.float32)
        rows = (2 if kind == 0 else 1) * d_in
        W = (rng.standard_normal((rows, d_out)) / np.sqrt(rows)).astype(np.float32)
        b = rng.standard_normal(d_out).astype(np.float32)
        relu = layer < L
        ld = gnnv.layer_desc(d_in, d_out, s_in, kind, aggr, 1 if relu else 0, prec)
        view = blocks.info(sync=False)[h]
        cap_dst, cap_src = view.max_dst, view.max_src
        dH, dW_, db_ = padded(Hsrc, cap_src), dev_f32(W), dev_f32(b)
        so = row_stride(d_out)
        Hdst = torch.full((cap_dst, so), float("nan"), device="cuda")
        A = torch.full((cap_dst, row_stride(d_in)), float("nan"), device="cuda")
        gnnv.layer_fwd(blocks, layer, ld, dH, dW_, db_, Hdst, A)
        torch.cuda.synchronize()
        Ho, Ao = layer_fwd(ob, Hsrc[:, :d_in], W, b, relu, kname, aname)
        Hm, Am = layer_fwd(ob, Hsrc[:, :d_in], W, b, relu, kname, aname, absval=True)
        Hg, Ag = Hdst[: ob.n_dst].cpu().numpy(), A[: ob.n_dst].cpu().numpy()
        assert torch.isnan(Hdst[ob.n_dst:]).all() and torch.isnan(A[ob.n_dst:]).all()  # rows >= n_dst untouched
        assert_close_cond(Ag[:, :d_in], Ao, Am, RTOL32, f"A layer {layer}")
        assert (Ag[:, d_in:] == 0).all() and (Hg[:, d_out:] == 0).all()
        assert_close_cond(Hg[:, :d_out], Ho, Hm, rtol, f"H layer {layer}")
        # backward with a random upstream gradient
        G = np.zeros((ob.n_dst, so), np.float32)
        G[:, :d_out] = rng.standard_normal((ob.n_dst, d_out)).astype(np.float32)
        need_dx = layer > 1
        Gsrc = torch.full((cap_src, s_in), float("nan"), device="cuda") if need_dx else None
        dW = torch.full((rows, d_out), float("nan"), device="cuda")
        db = torch.full((d_out,), float("nan"), device="cuda")
        gnnv.layer_bwd(blocks, layer, ld, padded(G, cap_dst), Hdst, dH, A, dW_, Gsrc, dW, db)
        torch.cuda.synchronize()
        if need_dx:
            Gsrc = Gsrc[: ob.n_src]
        # oracle backward on the GPU's forward values (same ReLU mask)
        rW, rb, rX = layer_bwd(ob, Hsrc[:, :d_in], Ag[:, :d_in], Hg[:, :d_out], W, G[:, :d_out], relu, need_dx,
                               kname, aname)
        mW, mb, mX = layer_bwd(ob, np.abs(Hsrc[:, :d_in]), np.abs(Ag[:, :d_in]), Hg[:, :d_out], np.abs(W),
                               np.abs(G[:, :d_out]), relu, need_dx, kname, aname)
        assert_close_cond(dW.cpu().numpy(), rW, mW, rtol, f"dW layer {layer}")
        assert_close_cond(db.cpu().numpy(), rb, mb, rtol, f"db layer {layer}")
        if need_dx:
            gx = Gsrc.cpu().numpy()
            assert_close_cond(gx[:, :d_in], rX, mX, rtol, f"dHsrc layer {layer}")
            assert (gx[:, d_in:] == 0).all()


def test_ce_loss_parity(mini):
    gd, g = mini
    seeds = epoch_seeds(gd.n, 0)[:333]
    blocks, hb = gpu_sample(g, seeds, [4], 1)
    C = gd.C
    so = row_stride(C)
    z = np.zeros((len(seeds), so), np.float32)
    z[:, :C] = 3 * np.random.default_rng(1).standard_normal((len(seeds), C))
    loss = torch.zeros(1, device="cuda")
    dz = torch.full((len(seeds), so), float("nan"), device="cuda")
    gnnv.ce_loss(blocks, g, dev_f32(z), C, so, 1000, loss, dz)
    torch.cuda.synchronize()
    rl, rdz = ce_loss(z[:, :C], gd.labels[seeds], 1000)
    assert abs(float(loss.item()) - rl) <= 1e-5 * abs(rl)
    dzg = dz.cpu().numpy()
    np.testing.assert_allclose(dzg[:, :C], rdz, rtol=1e-5, atol=1e-9)
    assert (dzg[:, C:] == 0).all()
    # deterministic: same result twice, bitwise
    loss2 = torch.zeros(1, device="cuda")
    gnnv.ce_loss(blocks, g, dev_f32(z), C, so, 1000, loss2, dz)
    torch.cuda.synchronize()
    assert loss.item() == loss2.item()


# -------------------------------------------------------------- full step
@pytest.mark.parametrize("kind,prec", [(0, 0), (1, 0), (0, 1), (0, 2), (1, 2)])
def test_step_parity(mini, kind, prec):
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    kname = "sage" if kind == 0 else "gcn"
    w = init_weights(dims, kind=kname)
    cache = gnnv.Cache(g, cfg["ratio"])
    tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], cfg["batch"], w, kind=kind, prec=prec)
    perm = epoch_seeds(gd.n, 0)
    seeds = perm[: cfg["batch"]]
    lr = 0.05
    loss, tm = tr.step(seeds, len(seeds), 2 * len(seeds), 0x5EED, lr, timing=True)
    ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, cfg["fanouts"], 0x5EED, w, lr,
                     n_global=2 * len(seeds), kind=kname)
    tol = {0: 1e-4, 1: 2e-2, 2: 5e-3}[prec]
    assert abs(loss - ref["loss"]) <= tol * abs(ref["loss"])
    grads = gnnv.unflat_params(tr.grads(), dims, kind)
    if prec == 0:
        for i, ((gW, gb), (rW, rb)) in enumerate(zip(grads, ref["grads"])):
            assert normwise(gW, rW) < tol, (i, normwise(gW, rW))
            assert normwise(gb, rb) < tol, (i, normwise(gb, rb))
        newp = gnnv.unflat_params(tr.params(), dims, kind)
        for (pW, pb), (nW, nb) in zip(newp, ref["new_weights"]):
            assert normwise(pW, nW) < 1e-5
    else:
        # bf16 (reading Q18): each layer of the step's forward chain vs the
        # oracle fed the GPU's own input (condition-aware 2e-2).  Gradients are
        # compared by direction: bf16 rounding flips the ReLU mask of
        # pre-activations within ~2^-8 of zero, so a masked gradient differs by
        # 100% on those elements and a normwise bound is ill-posed.
        # (with the tf32 SAGE trainer's fused L2 push: layer 2 on the GPU's
        # [H^1_dst | A^2], A^2 against the oracle's layer 1, gpu_util)
        hb = blocks_to_host(tr.blocks)
        check_forward_chain(tr, hb, dims, w, RTOL[prec], "step", kind=kname, max_rows=10**9)
        for i, ((gW, gb), (rW, rb)) in enumerate(zip(grads, ref["grads"])):
            for a_, b_ in ((gW, rW), (gb, rb)):
                cos = float(np.dot(a_.ravel(), b_.ravel()) / (np.linalg.norm(a_) * np.linalg.norm(b_) + 1e-30))
                assert cos > 0.98, (i, cos)
    st = tr.stats()
    slot, owner, _ = cache_slots(gd.indptr, cfg["ratio"])
    cnt = access_counts(slot, owner, ref["frontiers"][-1])
    assert st.tolist() == [cnt["rows"], cnt["hits_local"], cnt["hits_peer"], cnt["misses_host"]]
    assert all(v >= 0 for v in tm.values())
    # second step from the updated weights keeps matching
    seeds2 = perm[cfg["batch"]: 2 * cfg["batch"]]
    loss2, _ = tr.step(seeds2, len(seeds2), len(seeds2), 0x5EED + 1, lr)
    ref2 = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds2, cfg["fanouts"], 0x5EED + 1,
                      ref["new_weights"], lr, kind=kname)
    assert abs(loss2 - ref2["loss"]) <= tol * abs(ref2["loss"])


def test_step_device_seeds_and_errors(mini):
    gd, g = mini
    dims = [gd.d, 32, gd.C]
    w = init_weights(dims)
    cache = gnnv.Cache(g, 0.5)
    tr = gnnv.Trainer(g, cache, dims, [5, 5], 128, w)
    seeds = epoch_seeds(gd.n, 3)[:128]
    l1, _ = tr.step(dev_i32(seeds), 128, 128, 9, 0.0, on_host=False)
    l2, _ = tr.step(seeds, 128, 128, 9, 0.0, on_host=True)
    assert l1 == l2  # lr 0: identical iteration, bitwise
    with pytest.raises(gnnv.GnnvError):
        tr.step(np.array([1, 1, 2], np.int32), 3, 3, 9, 0.0)
    with pytest.raises(gnnv.GnnvError):
        tr.step(seeds, 129, 129, 9, 0.0)
    l3, _ = tr.step(seeds, 128, 128, 9, 0.0)
    assert l3 == l1


def test_device_seed_out_of_range(mini):
    """DEVICE seeds are range-checked on the device (host seeds on the host):
    an id outside [0, N) makes the step report PARAM at its sync point, no
    kernel reads out of bounds (the id is replaced by vertex 0), the SGD
    update of that step is skipped, and the flag does not outlive the batch
    -- the next valid step (also through the asynchronous loss ring)
    succeeds."""
    gd, g = mini
    dims = [gd.d, 32, gd.C]
    cache = gnnv.Cache(g, 0.5)
    tr = gnnv.Trainer(g, cache, dims, [5, 5], 128, init_weights(dims))
    seeds = epoch_seeds(gd.n, 3)[:128]
    p0 = tr.params().copy()
    for bad_id in (gd.n, -7, 2**31 - 1):
        bad = seeds.copy()
        bad[17] = bad_id
        with pytest.raises(gnnv.GnnvError) as e:
            tr.step(dev_i32(bad), 128, 128, 9, 0.1, on_host=False)
        assert e.value.status == gnnv.ERR_PARAM
        np.testing.assert_array_equal(tr.params(), p0)  # the bad batch was not applied
    # asynchronous path: the bad step's ticket reports PARAM, the next one is clean
    tr.step(dev_i32(bad), 128, 128, 9, 0.1, on_host=False, want_loss=False)
    t_bad = tr.loss_async()
    tr.step(dev_i32(seeds), 128, 128, 9, 0.0, on_host=False, want_loss=False)
    t_ok = tr.loss_async()
    with pytest.raises(gnnv.GnnvError):
        tr.loss_result(t_bad)
    assert np.isfinite(tr.loss_result(t_ok))
    l_ok, _ = tr.step(dev_i32(seeds), 128, 128, 9, 0.0, on_host=False)
    assert np.isfinite(l_ok)
    np.testing.assert_array_equal(tr.params(), p0)
    tr.free()


@pytest.mark.parametrize("prec", [0, 1, 2])
@pytest.mark.parametrize("d_in,d_out,kind", [(1433, 256, 0), (256, 256, 0), (256, 47, 0), (602, 41, 0),
                                             (128, 40, 1), (100, 256, 0), (7, 13, 0), (256, 172, 1)])
def test_layer_shapes(mini, prec, d_in, d_out, kind):
    """GEMM shape sweep (all config widths, ragged K/N, both precisions) on a
    real sampled block; layer 2 of the mini blocks (so dX is exercised)."""
    gd, g = mini
    seeds = epoch_seeds(gd.n, 5)[:257]
    blocks, hb = gpu_sample(g, seeds, [7, 6], 21, max_seeds=512)
    layer, L = 2, 2
    ob = _oracle_block(hb, L - layer)
    rng = np.random.default_rng(d_in * 7 + d_out)
    s_in = row_stride(d_in)
    Hsrc = np.zeros((ob.n_src, s_in), np.float32)
    Hsrc[:, :d_in] = rng.standard_normal((ob.n_src, d_in)).astype(np.float32)
    rows = (2 if kind == 0 else 1) * d_in
    W = (rng.standard_normal((rows, d_out)) / np.sqrt(rows)).astype(np.float32)
    b = rng.standard_normal(d_out).astype(np.float32)
    kname = "sage" if kind == 0 else "gcn"
    ld = gnnv.layer_desc(d_in, d_out, s_in, kind, 0, 1, prec)
    so = row_stride(d_out)
    view = blocks.info(sync=False)[L - layer]
    cap_dst, cap_src = view.max_dst, view.max_src
    dH, dW_, db_ = padded(Hsrc, cap_src), dev_f32(W), dev_f32(b)
    Hdst = torch.full((cap_dst, so), float("nan"), device="cuda")
    A = torch.full((cap_dst, s_in), float("nan"), device="cuda")
    gnnv.layer_fwd(blocks, layer, ld, dH, dW_, db_, Hdst, A)
    torch.cuda.synchronize()
    rtol = RTOL[prec]
    Ho, Ao = layer_fwd(ob, Hsrc[:, :d_in], W, b, True, kname)
    Hm, _ = layer_fwd(ob, Hsrc[:, :d_in], W, b, True, kname, absval=True)
    Hg, Ag = Hdst[: ob.n_dst].cpu().numpy(), A[: ob.n_dst].cpu().numpy()
    assert_close_cond(Hg[:, :d_out], Ho, Hm, rtol, "H")
    assert (Hg[:, d_out:] == 0).all()
    assert torch.isnan(Hdst[ob.n_dst:]).all()
    G = np.zeros((ob.n_dst, so), np.float32)
    G[:, :d_out] = rng.standard_normal((ob.n_dst, d_out)).astype(np.float32)
    Gsrc = torch.full((cap_src, s_in), float("nan"), device="cuda")
    dW = torch.full((rows, d_out), float("nan"), device="cuda")
    db = torch.full((d_out,), float("nan"), device="cuda")
    gnnv.layer_bwd(blocks, layer, ld, padded(G, cap_dst), Hdst, dH, A, dW_, Gsrc, dW, db)
    torch.cuda.synchronize()
    Gsrc = Gsrc[: ob.n_src]
    rW, rb, rX = layer_bwd(ob, Hsrc[:, :d_in], Ag[:, :d_in], Hg[:, :d_out], W, G[:, :d_out], True, True, kname)
    mW, mb, mX = layer_bwd(ob, np.abs(Hsrc[:, :d_in]), np.abs(Ag[:, :d_in]), Hg[:, :d_out], np.abs(W),
                           np.abs(G[:, :d_out]), True, True, kname)
    assert_close_cond(dW.cpu().numpy(), rW, mW, rtol, "dW")
    assert_close_cond(db.cpu().numpy(), rb, mb, rtol, "db")
    gx = Gsrc.cpu().numpy()
    assert_close_cond(gx[:, :d_in], rX, mX, rtol, "dHsrc")
    assert (gx[:, d_in:] == 0).all()


def test_pipelined_steps_match_sequential(mini):
    """Eq.4 pipeline: prefetching sample+gather of step t+1 on the side stream
    changes nothing in the results (the first loss bitwise, the rest and the
    parameters to the rounding of the atomic backward)."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    w = init_weights(dims)
    cache = gnnv.Cache(g, cfg["ratio"])
    B = cfg["batch"]
    perm = epoch_seeds(gd.n, 0)
    batches = [perm[i * B:(i + 1) * B] for i in range(5)]
    seq = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, w, prec=2)
    l_seq = [seq.step(bt, B, B, 100 + i, 0.05)[0] for i, bt in enumerate(batches)]
    pip = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, w, prec=2)
    pip.prefetch(batches[0], B, 100)
    l_pip = []
    for i, bt in enumerate(batches):
        pip.step(bt, B, B, 100 + i, 0.05, want_loss=False)
        if i + 1 < len(batches):
            pip.prefetch(batches[i + 1], B, 101 + i)
        l_pip.append(pip.read_loss())
    assert l_seq[0] == l_pip[0]
    # later steps differ by the atomic summation order of the backward's
    # repeated src ids: fp32 rounding, or bf16 rounding for the tf32
    # trainer's bf16 dL/dH^1 (reading Q30)
    bf16 = seq.bf16act()
    np.testing.assert_allclose(l_pip, l_seq, rtol=1e-4 if bf16 else 1e-5)
    assert normwise(pip.params(), seq.params()) < (5e-4 if bf16 else 1e-5)
    with pytest.raises(gnnv.GnnvError):  # one pending prefetch at a time
        pip.prefetch(batches[0], B, 7)
        pip.prefetch(batches[1], B, 8)

    # device seeds, prefetches ordered on their own stream, no host sync
    # between steps: the overlapped schedule still yields the same losses
    import torch
    dev = torch.as_tensor(np.concatenate(batches)).cuda()
    torch.cuda.synchronize()
    pf = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    dv = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, w, prec=2)
    losses = []
    dv.prefetch(dev[0:B].data_ptr(), B, 100, on_host=False, stream=pf)
    for i in range(len(batches)):
        dv.step(dev[i * B:(i + 1) * B].data_ptr(), B, B, 100 + i, 0.05, on_host=False, want_loss=False,
                stream=main)
        if i + 1 < len(batches):
            dv.prefetch(dev[(i + 1) * B:(i + 2) * B].data_ptr(), B, 101 + i, on_host=False, stream=pf)
        losses.append(dv.read_loss(stream=main))
    np.testing.assert_allclose(losses, l_seq, rtol=1e-4 if bf16 else 1e-5)
    assert normwise(dv.params(), seq.params()) < (5e-4 if bf16 else 1e-5)


# ------------------------------------------- locality-biased sampling (NEXT-2)
@pytest.mark.parametrize("bias", [0.25, 0.5, 1.0])
@pytest.mark.parametrize("fan", [[15, 10, 5], [5, 3], [32, 2]])
def test_biased_sampling_bit_exact(mini, bias, fan):
    gd, g = mini
    cache = gnnv.Cache(g, 0.3)
    slot, _, _ = cache_slots(gd.indptr, 0.3)
    seeds = epoch_seeds(gd.n, 1)[:300]
    blocks = gnnv.Blocks(g, 512, fan)
    blocks.set_locality(cache, bias)
    blocks.sample(dev_i32(seeds), len(seeds), 77)
    hb = blocks_to_host(blocks)
    oF, oB = sample_blocks(gd.indptr, gd.indices, seeds, fan, 77, slot >= 0, bias)
    assert_blocks_equal(hb, oF, oB)


def test_biased_trainer_raises_hit_rate(mini):
    """The trainer's locality knob: blocks equal the oracle's biased blocks,
    and the host-miss count falls as the bias grows (the point of NEXT-2)."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    cache = gnnv.Cache(g, 0.2)
    slot, owner, _ = cache_slots(gd.indptr, 0.2)
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    misses = []
    for bias in (0.0, 0.5, 1.0):
        tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], cfg["batch"], init_weights(dims), prec=2)
        tr.set_locality(bias)
        tr.step(seeds, len(seeds), len(seeds), 5, 0.01)
        oF, oB = sample_blocks(gd.indptr, gd.indices, seeds, cfg["fanouts"], 5, slot >= 0, bias)
        assert_blocks_equal(blocks_to_host(tr.blocks), oF, oB)
        cnt = access_counts(slot, owner, oF[-1])
        st = tr.stats().tolist()
        assert st == [cnt["rows"], cnt["hits_local"], cnt["hits_peer"], cnt["misses_host"]]
        misses.append(st[3] / st[0])
        tr.free()
    assert misses[0] > misses[1] > misses[2], misses
    tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], cfg["batch"], init_weights(dims), prec=2)
    for bad in (0.3, -0.25, 1.25):  # the library validates the bias itself (1 + 4b must be an integer in 1..5)
        with pytest.raises(gnnv.GnnvError):
            tr.set_locality(bad)
    tr.free()


# ------------------------------------------------- dynamic cache (NEXT-3)
@pytest.mark.parametrize("policy", [2, 3])  # FIFO, LRU
@pytest.mark.parametrize("ratio", [0.1, 0.01])
def test_dynamic_cache_bit_exact(mini, policy, ratio):
    """Batch after batch: gathered rows (hits now come from rows the cache
    admitted earlier), the slot map, the slot owners and the cumulative
    (hits, misses, replaced, admitted) equal the oracle's sequential
    simulation of SPEC's access_batch."""
    from gpu_util import read_i32
    from oracle.cache import DynamicCache

    gd, g = mini
    fan = [10, 5]
    cache = gnnv.Cache(g, ratio, policy=policy)
    C = int(np.floor(ratio * gd.n))
    ref = DynamicCache(gd.n, C, policy)
    perm = epoch_seeds(gd.n, 2)
    blocks = gnnv.Blocks(g, 400, fan)
    for t in range(6):
        seeds = perm[(t % 3) * 400:(t % 3 + 1) * 400]  # batches repeat: later ones hit admitted rows
        blocks.sample(dev_i32(seeds), len(seeds), 40 + (t % 3))
        views = blocks.info()
        X = torch.empty((views[-1].max_src, gd.stride), dtype=torch.float32, device="cuda")
        stats = torch.zeros(4, dtype=torch.int64, device="cuda")
        gnnv.gather(cache, blocks, X, stats)
        cache.update(blocks, X)
        torch.cuda.synchronize()
        FL = blocks_to_host(blocks)[-1][4]
        assert X[: len(FL)].cpu().numpy().tobytes() == oracle.gather_rows(gd.feats, FL).tobytes()
        out = ref.access_batch(FL)
        s = stats.cpu().tolist()
        assert s[0] == out["rows"] and s[1] == out["hits"] and s[3] == out["misses"], (t, s, out)
        np.testing.assert_array_equal(read_i32(cache.info().d_slot, gd.n), ref.slot)
        if C:
            np.testing.assert_array_equal(read_i32(cache.owners_ptr(), C), ref.owner)
        assert cache.counters().tolist() == [ref.hits, ref.misses, ref.replaced, ref.misses if C else 0]


def test_dynamic_cache_trainer_pipelined(mini):
    """The trainer admits each batch's misses after its gather (also when
    the gather is a prefetch on the side stream): per-step hit counters equal
    the oracle's sequence."""
    from oracle.cache import DynamicCache

    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    B = cfg["batch"]
    cache = gnnv.Cache(g, 0.1, policy=3)
    ref = DynamicCache(gd.n, int(np.floor(0.1 * gd.n)), 3)
    tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, init_weights(dims), prec=2)
    perm = epoch_seeds(gd.n, 0)
    batches = [perm[(i % 2) * B:(i % 2 + 1) * B] for i in range(5)]
    tr.prefetch(batches[0], B, 200)
    for i in range(5):
        tr.step(batches[i], B, B, 200 + i, 0.01, want_loss=False)
        st = tr.stats().tolist()  # this step's batch (the stats of its buffer set)
        if i + 1 < 5:
            tr.prefetch(batches[i + 1], B, 201 + i)
        tr.read_loss()
        oF, _ = sample_blocks(gd.indptr, gd.indices, batches[i], cfg["fanouts"], 200 + i)
        out = ref.access_batch(oF[-1])
        assert st == [out["rows"], out["hits"], 0, out["misses"]], (i, st, out)
    tr.free()
    torch.cuda.synchronize()
    assert cache.counters().tolist()[:3] == [ref.hits, ref.misses, ref.replaced]


def test_dynamic_cache_serial_then_prefetch(mini):
    """a serial step's admission must be ordered before a
    following prefetch's gather + admission (the prefetch runs on the
    trainer's side stream).  step, prefetch, step, step(serial), prefetch,
    step with an LRU cache: per-step counters equal the oracle's sequence."""
    from oracle.cache import DynamicCache

    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    B = cfg["batch"]
    cache = gnnv.Cache(g, 0.1, policy=3)
    ref = DynamicCache(gd.n, int(np.floor(0.1 * gd.n)), 3)
    tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, init_weights(dims), prec=2)
    perm = epoch_seeds(gd.n, 0)
    batches = [perm[(i % 3) * B:(i % 3 + 1) * B] for i in range(5)]
    other = torch.cuda.Stream()  # host seeds: no stream dependency at all
    plan = ["serial", "prefetched", "serial", "serial", "prefetched"]
    for i, how in enumerate(plan):
        if how == "prefetched":
            tr.prefetch(batches[i], B, 300 + i, on_host=True, stream=other)
        tr.step(batches[i], B, B, 300 + i, 0.01, want_loss=False)
        st = tr.stats().tolist()
        oF, _ = sample_blocks(gd.indptr, gd.indices, batches[i], cfg["fanouts"], 300 + i)
        out = ref.access_batch(oF[-1])
        assert st == [out["rows"], out["hits"], 0, out["misses"]], (i, how, st, out)
    tr.free()
    torch.cuda.synchronize()
    assert cache.counters().tolist()[:3] == [ref.hits, ref.misses, ref.replaced]


def test_nccl_comm_world1(mini):
    """The NCCL plumbing of the data-parallel path on one rank: the library
    loads NCCL, creates a communicator from a unique id, runs the trainer's
    all-reduce (identity for one rank) and builds a SHARDED cache with it."""
    gd, g = mini
    comm = gnnv.Comm(0, 1, gnnv.Comm.unique_id(), 0)
    t = torch.arange(10, dtype=torch.float32, device="cuda")
    comm.allreduce_sum(t)
    torch.cuda.synchronize()
    assert t.tolist() == list(range(10))
    cache = gnnv.Cache(g, 0.3, placement=gnnv.PLACE_SHARDED, comm=comm)
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], cfg["batch"], init_weights(dims), prec=2, comm=comm)
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    loss, _ = tr.step(seeds, len(seeds), len(seeds), 3, 0.01)
    ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, cfg["fanouts"], 3, init_weights(dims),
                     0.01)
    assert abs(loss - ref["loss"]) <= 5e-3 * abs(ref["loss"])
    tr.free()
    cache.free()
    comm.free()


def test_async_loss_readback(mini):
    """gnnv_trainer_loss_async / _loss_result return the same losses as the
    synchronous read, with several steps in flight."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    B = cfg["batch"]
    perm = epoch_seeds(gd.n, 0)
    cache = gnnv.Cache(g, 0.3)
    a = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, init_weights(dims), prec=2)
    b = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, init_weights(dims), prec=2)
    # lr 0: every step's loss is then a deterministic function of its batch
    # (the backward's atomic order cannot reach the next step's weights)
    sync = [a.step(perm[i * B:(i + 1) * B], B, B, 50 + i, 0.0)[0] for i in range(10)]
    tickets = []
    for i in range(10):
        b.step(perm[i * B:(i + 1) * B], B, B, 50 + i, 0.0, want_loss=False)
        tickets.append(b.loss_async())
    got = [b.loss_result(t) for t in tickets[-8:]]
    assert got == sync[-8:]
    with pytest.raises(gnnv.GnnvError):
        b.loss_result(tickets[0])  # recycled (ring of 8)


@pytest.mark.parametrize("kind", ["sage", "gcn"])
@pytest.mark.parametrize("prec", [0, 2])
def test_step_degenerate_graph(kind, prec):
    """A whole training step on a graph with an isolated seed (zero sampled
    neighbours: mean aggregate 0 for SAGE, the vertex itself for GCN --
    reading Q15) and rows with fewer neighbours than the fanout, as fp32 and
    as tf32 with the whole table cached (the layer-1 table-reading path)."""
    lib()
    gd = tiny_graph("isolated", d=6, C=3)
    g = gnnv.Graph.from_data(gd)
    dims = [gd.d, 8, gd.C]
    kid = gnnv.KIND_SAGE if kind == "sage" else gnnv.KIND_GCN
    w = init_weights(dims, kind=kind)
    cache = gnnv.Cache(g, 1.0)
    tr = gnnv.Trainer(g, cache, dims, [3, 2], 4, w, kind=kid, prec=prec)
    seeds = np.array([5, 0, 2, 4])  # 5 is isolated
    loss, _ = tr.step(seeds, 4, 4, 17, 0.1)
    ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, [3, 2], 17, w, 0.1, kind=kind)
    tol = 1e-4 if prec == 0 else 5e-3
    assert abs(loss - ref["loss"]) <= tol * abs(ref["loss"])
    grads = gnnv.unflat_params(tr.grads(), dims, kid)
    for (gW, gb), (rW, rb) in zip(grads, ref["grads"]):
        assert normwise(gW, rW) < (1e-4 if prec == 0 else 2e-2)
        assert normwise(gb, rb) < (1e-4 if prec == 0 else 2e-2)


def test_step_whole_table_gather4(mini, option):
    """Whole table cached, tf32 SAGE: the layer-1 GEMMs (forward and dW) read
    H_dst straight from the degree-ordered table with TMA gather4 through the
    gather's row indices and X is never written (x_level -1).  The forward
    reads exactly the values the materialised path reads, in the same order,
    (GNNV_XROWS=1), so the loss equals bit for bit that of the same step with X materialised
    (a cache one row short of the table: ratio (N-1)/N); the gradients match
    it to the backward's atomic summation order.  Both match the oracle."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    w = init_weights(dims)
    L = len(cfg["fanouts"])
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    out = {}
    option("GNNV_XROWS", 1)  # read when a trainer is created
    option("GNNV_NO_BF16ACT", 1)  # fp32 intermediates: the two paths then agree to fp32 atomic rounding
    option("GNNV_NO_BF16TABLE", 1)  # and the whole-table path aggregates the fp32 table, as X's copy does
    for name, ratio in (("rows", 1.0), ("copy", (gd.n - 1) / gd.n)):
        tr = gnnv.Trainer(g, gnnv.Cache(g, ratio), dims, cfg["fanouts"], cfg["batch"], w, prec=gnnv.PREC_TF32)
        loss, _ = tr.step(seeds, len(seeds), len(seeds), 0x5EED, 0.05)
        out[name] = (loss, tr.grads(), tr.x_level(), tr)
    assert out["rows"][2] == -1 and out["copy"][2] == L
    assert out["rows"][0] == out["copy"][0], (out["rows"][0], out["copy"][0])
    assert normwise(out["rows"][1], out["copy"][1]) < 2e-5  # fp32 atomic-order rounding of the backward
    ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, cfg["fanouts"], 0x5EED, w, 0.05)
    assert abs(out["rows"][0] - ref["loss"]) <= 5e-3 * abs(ref["loss"])
    tr = out["rows"][3]
    pr, _ = tr.rowidx()
    slot, _, _ = cache_slots(gd.indptr, 1.0)
    FL = ref["frontiers"][-1]
    np.testing.assert_array_equal(read_i32(pr, len(FL)), slot[FL])
    # layer 1's output vs the oracle fed the exact feature rows
    hb = blocks_to_host(tr.blocks)
    ob = _oracle_block(hb, L - 1)
    Hin = oracle.gather_rows(gd.feats, FL)[:, : dims[0]]
    p_out, s_out = tr.activation(1)
    n_keep = hb[L - 2][0] if tr.l2push() else ob.n_dst  # fused push: H^1 stored for layer 2's dst prefix only
    Hout = read_f32(p_out, n_keep, s_out)[:, : dims[1]]
    blk, Hs = sub_block(ob, Hin, np.arange(n_keep))
    Ho, _ = layer_fwd(blk, Hs, w[0][0], w[0][1], True)
    Hm, _ = layer_fwd(blk, Hs, w[0][0], w[0][1], True, absval=True)
    assert_close_cond(Hout, Ho, Hm, RTOL[2], "layer 1 (gather4 H_dst)")


def test_dynamic_tile_scheduler_bitwise_neutral(mini, option):
    """The persistent tf32 fwd/dX GEMMs claim their tiles from a device
    counter (a CTA that starts late takes fewer tiles); which CTA computes a
    tile does not change its arithmetic, so a whole pipelined step's forward -- loss
    and every activation -- is bitwise the static round
    robin's (GNNV_STATIC_TILES), also for ragged tile counts, over repeated
    steps (the scheduler slots reset themselves)."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, 96, 80, gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    perm = epoch_seeds(gd.n, 0)
    out = {}
    for name in ("dynamic", "static"):
        option("GNNV_STATIC_TILES", 1 if name == "static" else 0)
        tr = gnnv.Trainer(g, gnnv.Cache(g, 0.3), dims, cfg["fanouts"], cfg["batch"], w, prec=gnnv.PREC_TF32)
        res = []
        for t in range(3):
            seeds = perm[t * 300:(t + 1) * 300]
            tr.prefetch(seeds, len(seeds), 40 + t)
            loss, _ = tr.step(seeds, len(seeds), len(seeds), 40 + t, 0.0)
            hb = blocks_to_host(tr.blocks)
            acts = [loss]
            for lvl in range(1, L + 1):
                acts.append(read_activation(tr, lvl, hb[L - lvl][0]).tobytes())
            res.append(acts)
        out[name] = res
        tr.free()
    assert out["dynamic"] == out["static"]


@pytest.mark.parametrize("ratio", [0.3, 1.0])
def test_bf16_intermediates(mini, option, ratio):
    """The tf32 SAGE trainer (default; GNNV_NO_BF16ACT=1: off) keeps H^1 and dL/dH^1 (the widest
    activations, L = 3) as bf16 -- the layer-2 aggregation reads the bf16
    copy, layer 1's dW reads the bf16 gradient.  The step against the oracle
    at the tf32 bounds (gpu_util chain checks: A^2 exact over the bf16
    values, layer 2 on the GPU's own inputs, every dW/db through the
    oracle's backward chain), and against the fp32-intermediate step: loss
    within 2e-3, gradient directions within cos 0.999."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    w = init_weights(dims)
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    B = len(seeds)
    out = {}
    for name in ("bf16", "fp32"):
        option("GNNV_NO_BF16ACT", 0 if name == "bf16" else 1)
        tr = gnnv.Trainer(g, gnnv.Cache(g, ratio), dims, cfg["fanouts"], cfg["batch"], w, prec=gnnv.PREC_TF32)
        assert tr.bf16act() == (name == "bf16")
        if name == "bf16":
            fwd16 = tr.fwd16()
        tr.prefetch(seeds, B, 0x5EED)
        loss, _ = tr.step(seeds, B, B, 0x5EED, 0.0)
        grads = gnnv.unflat_params(tr.grads(), dims)
        if name == "bf16":
            hb = blocks_to_host(tr.blocks)
            L = len(cfg["fanouts"])
            X0 = oracle.gather_rows(gd.feats, hb[L - 1][4])[:, : dims[0]] if tr.x_level() < L else None
            H, Aagg, blks = check_forward_chain(tr, hb, dims, w, RTOL[2], "bf16act", X0=X0, max_rows=10**9)
            check_backward_chain(tr, blks, H, Aagg, dims, w, grads, gd.labels[seeds], B, RTOL[2], "bf16act")
        out[name] = (loss, grads)
        tr.free()
    (lb, gb_), (lf, gf) = out["bf16"], out["fp32"]
    assert abs(lb - lf) <= 2e-3 * abs(lf), (lb, lf)
    # with the whole table cached layer 1's GEMMs also run over bf16 copies
    # (readings Q32/Q33): ReLU decisions near 0 flip between the runs, so
    # the cross-run direction bound is wider there (the per-layer chain
    # checks above hold at the tf32 bounds either way)
    bound = 0.995 if fwd16 else 0.999
    coss = []
    for (aW, ab), (bW, bb) in zip(gb_, gf):
        for a_, b_ in ((aW, bW), (ab, bb)):
            coss.append(float(np.dot(a_.ravel(), b_.ravel()) / (np.linalg.norm(a_) * np.linalg.norm(b_) + 1e-30)))
    assert min(coss) > bound, coss


def test_bf16_table_layer1_aggregation(mini, option):
    """Whole table cached, tf32 SAGE: layer 1 aggregates the cache's bf16
    copy of the table (reading Q31; the gathered rows stay the exact fp32
    ones).  A^1 against the fp32 aggregation of the bf16-rounded feature
    rows (1e-5) and of the exact rows (bf16 rounding, 2^-8 of |.|); the
    step's loss within 1e-3 of the fp32-table step."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    B = len(seeds)
    losses = {}
    option("GNNV_NO_FWD16", 1)  # the layer-1 GEMM stays TF32: only the aggregation's source differs
    for name in ("bf16", "fp32"):
        option("GNNV_NO_BF16TABLE", 0 if name == "bf16" else 1)
        tr = gnnv.Trainer(g, gnnv.Cache(g, 1.0), dims, cfg["fanouts"], B, w, prec=gnnv.PREC_TF32)
        assert tr.table16() == (name == "bf16")
        losses[name], _ = tr.step(seeds, B, B, 0x5EED, 0.0)
        if name == "bf16":
            hb = blocks_to_host(tr.blocks)
            ob = _oracle_block(hb, L - 1)
            pa, sa = tr.aggregate(1)
            A = read_f32(pa, ob.n_dst, sa)[:, : gd.d]
            X = oracle.gather_rows(gd.feats, hb[L - 1][4])[:, : gd.d].astype(np.float64)
            X16 = (np.asarray(X, np.float32).view(np.uint32) + 0x7FFF + ((np.asarray(X, np.float32).view(np.uint32) >> 16) & 1)) & 0xFFFF0000
            X16 = X16.astype(np.uint32).view(np.float32).astype(np.float64)  # round to nearest even, as the device
            P = agg_matrix(ob)
            assert_close_cond(A, P @ X16, P @ np.abs(X16), 1e-5, "A^1 over the bf16 rows")
            assert_close_cond(A, P @ X, P @ np.abs(X), 2.0 ** -8, "A^1 vs the exact rows")
        tr.free()
    assert abs(losses["bf16"] - losses["fp32"]) <= 1e-3 * abs(losses["fp32"])


@pytest.mark.parametrize("pipelined", [False, True], ids=["serial", "pipelined"])
def test_bf16_layer1_dw(mini, option, pipelined):
    """Layer 1's dW over bf16 MN-major operands (gemm_dw16, reading Q32):
    its operands are exactly the bf16 roundings of the step's own fp32 X dst
    prefix (with 1.0 in column d: the db column) and A^1, and dW / db equal
    [X16 | A16]^T G16 and colsum(G16) in fp64 up to fp32 accumulation
    (rtol 1e-5 of the |.| product).  A large batch first, then a smaller
    one: the second's ragged last k-block sits over rows the first step
    left non-zero, so a missing tail mask would show.  Against the TF32 dW
    (GNNV_NO_DW16=1): the same loss bitwise (the forward is unchanged), dW
    of layer 1 within cos 0.9999 and through the oracle's backward chain."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    perm = epoch_seeds(gd.n, 0)
    B = cfg["batch"]
    runs = {}
    option("GNNV_NO_FWD16", 1)  # the forward stays the TF32 one in both runs
    for name in ("dw16", "tf32"):
        option("GNNV_NO_DW16", 0 if name == "dw16" else 1)
        tr = gnnv.Trainer(g, gnnv.Cache(g, 1.0), dims, cfg["fanouts"], B, w, prec=gnnv.PREC_TF32)
        assert tr.dw16() == (name == "dw16") and not tr.fwd16()
        for t, n in ((0, B), (1, B // 3 + 7)):
            seeds = perm[t * B:t * B + n]
            if pipelined:
                tr.prefetch(seeds, n, 77 + t)
            loss, _ = tr.step(seeds, n, n, 77 + t, 0.0)
        grads = gnnv.unflat_params(tr.grads(), dims)
        if name == "dw16":
            hb = blocks_to_host(tr.blocks)
            ob = _oracle_block(hb, L - 1)
            M, d = ob.n_dst, gd.d
            px, pa, ld = tr.dw16_operands()
            X16 = read_bf16(px, M, ld)
            A16 = read_bf16(pa, M, ld)
            X_all = oracle.gather_rows(gd.feats, hb[L - 1][4])[:, :d]
            X = X_all[:M]
            np.testing.assert_array_equal(X16[:, :d], bf16_round(X))
            np.testing.assert_array_equal(X16[:, d], 1.0)
            p1, s1 = tr.aggregate(1)
            np.testing.assert_array_equal(A16[:, :d], bf16_round(read_f32(p1, M, s1)[:, :d]))
            pg, ldg = tr.gradient16(1)
            G16 = read_bf16(pg, M, ldg)[:, : dims[1]]
            Z = np.concatenate([X16[:, :d], A16[:, :d]], axis=1)
            assert_close_cond(grads[0][0], Z.T @ G16, np.abs(Z).T @ np.abs(G16), 1e-5, "dW^1 over the bf16 operands")
            assert_close_cond(grads[0][1], G16.sum(0), np.abs(G16).sum(0), 1e-5, "db^1 = colsum(G16)")
            H, Aagg, blks = check_forward_chain(tr, hb, dims, w, RTOL[2], "dw16",
                                                X0=X_all if tr.x_level() < L else None, max_rows=10**9)
            check_backward_chain(tr, blks, H, Aagg, dims, w, grads, gd.labels[seeds], n, RTOL[2], "dw16")
        runs[name] = (loss, grads)
        tr.free()
    assert runs["dw16"][0] == runs["tf32"][0]
    for a_, b_ in zip(runs["dw16"][1][0], runs["tf32"][1][0]):
        cos = float(np.dot(a_.ravel(), b_.ravel()) / (np.linalg.norm(a_) * np.linalg.norm(b_) + 1e-30))
        assert cos > 0.9999, cos


@pytest.mark.parametrize("pipelined", [False, True], ids=["serial", "pipelined"])
def test_bf16_layer1_fwd(mini, option, pipelined):
    """Layer 1's forward GEMM over the bf16 copies (kind::f16, reading Q33):
    Z = [X16 | A16] bf16(W) + b in fp64 is the reference -- the kept fp32
    rows of H^1 = relu(Z) within fp32 accumulation (rtol 1e-5 of the |.|
    product), every row of the bf16 copy within its own rounding (2^-8 of
    the |.| product); the whole step through the oracle's chains at the tf32
    bounds; loss within 2e-3 of the TF32 forward's (GNNV_NO_FWD16=1)."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    perm = epoch_seeds(gd.n, 0)
    B = cfg["batch"]
    losses = {}
    for name in ("fwd16", "tf32"):
        option("GNNV_NO_FWD16", 0 if name == "fwd16" else 1)
        tr = gnnv.Trainer(g, gnnv.Cache(g, 1.0), dims, cfg["fanouts"], B, w, prec=gnnv.PREC_TF32)
        assert tr.fwd16() == (name == "fwd16")
        for t, n in ((0, B), (1, B // 3 + 7)):
            seeds = perm[t * B:t * B + n]
            if pipelined:
                tr.prefetch(seeds, n, 91 + t)
            loss, _ = tr.step(seeds, n, n, 91 + t, 0.0)
        losses[name] = loss
        if name == "fwd16":
            hb = blocks_to_host(tr.blocks)
            M, d = hb[L - 1][0], gd.d
            px, pa, ld = tr.dw16_operands()
            Z16 = np.concatenate([read_bf16(px, M, ld)[:, :d], read_bf16(pa, M, ld)[:, :d]], axis=1)
            W0, b0 = w[0]
            W16 = bf16_round(W0)
            Z = Z16 @ W16 + b0.astype(np.float64)
            mag = np.abs(Z16) @ np.abs(W16) + np.abs(b0)
            keep = hb[L - 2][0]
            ph, sh = tr.activation(1)
            if ph:  # fp32 rows kept (not at L = 3 with the bf16 hidden-layer paths)
                H32 = read_f32(ph, keep, sh)[:, : dims[1]]
                assert_close_cond(H32, np.maximum(Z[:keep], 0), mag[:keep], 1e-5, "H^1 fp32 rows")
            p16, l16 = tr.activation16(1)
            H16 = read_bf16(p16, M, l16)[:, : dims[1]]
            assert_close_cond(H16, np.maximum(Z, 0), mag, 2.0 ** -8, "H^1 bf16 copy")
            grads = gnnv.unflat_params(tr.grads(), dims)
            X_all = oracle.gather_rows(gd.feats, hb[L - 1][4])[:, :d]
            H, Aagg, blks = check_forward_chain(tr, hb, dims, w, RTOL[2], "fwd16",
                                                X0=X_all if tr.x_level() < L else None, max_rows=10**9)
            check_backward_chain(tr, blks, H, Aagg, dims, w, grads, gd.labels[seeds], n, RTOL[2], "fwd16")
        tr.free()
    assert abs(losses["fwd16"] - losses["tf32"]) <= 2e-3 * abs(losses["tf32"]), losses


@pytest.mark.parametrize("hdw", [0, 1, 2], ids=["tf32dw", "bf16dw_conv", "bf16dw_tail"])
@pytest.mark.parametrize("ratio", [0.3, 1.0])
def test_bf16_hidden_layer_fwd(mini, option, ratio, hdw):
    """bf16 intermediates: layer 2's forward GEMM reads [bf16 H^1 dst prefix
    | bf16 A^2] (kind::f16, reading Q34) and its dW the same operands with a
    bf16 copy of its masked G.  A^2's bf16 copy is bit for bit the RNE
    rounding of the fp32 A^2 the aggregation also writes; H^2 equals
    relu([H16 | A16] bf16(W^2) + b^2) in fp64 to 1e-5 of the |.| product;
    dW^2 equals [H16 | A16]^T G16 to 1e-5, db^2 (summed from the fp32 G) the
    copy's column sums to its rounding;
    the forward and backward chains hold at the tf32 bounds; the loss is
    within 2e-3 of the TF32 layer-2 GEMM's (GNNV_NO_HID16=1)."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    B = len(seeds)
    losses = {}
    # layer 2's dW/dX: TF32 over fp32 G; over bf16 with G converted in the
    # dW call (opt-in GNNV_HID16_DW); over the fused output layer's bf16 G
    # and db partials (the default, GNNV_NO_TAIL16=0)
    option("GNNV_HID16_DW", 1 if hdw == 1 else 0)
    option("GNNV_NO_TAIL16", 0 if hdw == 2 else 1)
    for name in ("hid16", "tf32"):
        option("GNNV_NO_HID16", 0 if name == "hid16" else 1)
        tr = gnnv.Trainer(g, gnnv.Cache(g, ratio), dims, cfg["fanouts"], B, w, prec=gnnv.PREC_TF32)
        tr.prefetch(seeds, B, 0x5EED)
        losses[name], _ = tr.step(seeds, B, B, 0x5EED, 0.0)
        p16, ld = tr.aggregate16(2)
        assert bool(p16) == (name == "hid16")
        if name == "hid16":
            hb = blocks_to_host(tr.blocks)
            n2 = hb[L - 2][0]
            pa, sa = tr.aggregate(2)
            A32 = read_f32(pa, n2, sa)[:, : dims[1]]
            A16 = read_bf16(p16, n2, ld)[:, : dims[1]]
            np.testing.assert_array_equal(A16, bf16_round(A32))
            ph16, lh = tr.activation16(1)
            H16 = read_bf16(ph16, n2, lh)[:, : dims[1]]
            Xc = np.concatenate([H16, A16], axis=1)
            W2, b2 = w[1]
            W16 = bf16_round(W2)
            Z = Xc @ W16 + b2.astype(np.float64)
            mag = np.abs(Xc) @ np.abs(W16) + np.abs(b2)
            p2, s2 = tr.activation(2)
            H2 = read_f32(p2, n2, s2)[:, : dims[2]]
            assert_close_cond(H2, np.maximum(Z, 0), mag, 1e-5, "H^2 over the bf16 operands")
            grads = gnnv.unflat_params(tr.grads(), dims)
            pg, lg = tr.gradient16(2)
            assert bool(pg) == (hdw > 0) and tr.tail16() == (hdw == 2)
            if pg:  # layer 2's dW over the same operands and the bf16 copy of its (masked) G
                G16 = read_bf16(pg, n2, lg)[:, : dims[2]]
                assert_close_cond(grads[1][0], Xc.T @ G16, np.abs(Xc).T @ np.abs(G16), 1e-5, "dW^2 over bf16")
                assert_close_cond(grads[1][1], G16.sum(0), np.abs(G16).sum(0), 2.0 ** -8, "db^2 (fp32 G)")
            X0 = oracle.gather_rows(gd.feats, hb[L - 1][4])[:, : dims[0]] if tr.x_level() < L else None
            H, Aagg, blks = check_forward_chain(tr, hb, dims, w, RTOL[2], "hid16", X0=X0, max_rows=10**9)
            check_backward_chain(tr, blks, H, Aagg, dims, w, grads, gd.labels[seeds], B, RTOL[2], "hid16")
        tr.free()
    assert abs(losses["hid16"] - losses["tf32"]) <= 2e-3 * abs(losses["tf32"]), losses


@pytest.mark.parametrize("n", [1, 3, 33, 130])
def test_tiny_batches_bf16_paths(mini, n):
    """The whole-table TF32 trainer with every bf16 operand path on
    (readings Q30-Q34) at batch sizes that leave every tile ragged or empty
    (one seed: one row per layer-2 tile, a single k-block in the dW16 CTAs,
    most CTAs without chunks): the step against the oracle -- loss at the
    tf32 bound, every layer and dW/db through the oracle's chains."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    seeds = epoch_seeds(gd.n, 3)[:n]
    tr = gnnv.Trainer(g, gnnv.Cache(g, 1.0), dims, cfg["fanouts"], cfg["batch"], w, prec=gnnv.PREC_TF32)
    try:
        assert tr.dw16() and tr.fwd16() and tr.tail16()
        loss, _ = tr.step(seeds, n, n, 0xBEEF + n, 0.0)
        ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, cfg["fanouts"], 0xBEEF + n, w, 0.0)
        assert abs(loss - ref["loss"]) <= 5e-3 * abs(ref["loss"]), (loss, ref["loss"])
        hb = blocks_to_host(tr.blocks)
        grads = gnnv.unflat_params(tr.grads(), dims)
        X0 = oracle.gather_rows(gd.feats, hb[L - 1][4])[:, : dims[0]]
        H, Aagg, blks = check_forward_chain(tr, hb, dims, w, RTOL[2], f"tiny{n}", X0=X0, max_rows=10**9)
        check_backward_chain(tr, blks, H, Aagg, dims, w, grads, gd.labels[seeds], n, RTOL[2], f"tiny{n}")
    finally:
        tr.free()


@pytest.mark.parametrize("seeds", [[5], [5, 0, 2, 4], [0, 1, 2, 3]])
def test_last_hop_table_rows_degenerate(seeds):
    """The whole-table TF32 trainer's unrelabelled last hop (its CSR offsets
    a plain exclusive sum of the row counts) on a graph with an
    isolated vertex: a batch whose every hop is empty (seed 5 alone: no edge
    in any block, the closing offset 0), one mixing the isolated seed with
    rows of fewer neighbours than the fanout, and one without it; L = 3 so
    every bf16 operand path is on.  Serial and pipelined (Eq.4 prefetch)
    steps against the oracle: loss at the tf32 bound, every layer and dW/db
    through the oracle's chains."""
    lib()
    gd = tiny_graph("isolated", d=6, C=3)
    g = gnnv.Graph.from_data(gd)
    dims = [gd.d, 64, 64, gd.C]
    fan = [3, 2, 2]
    w = init_weights(dims)
    seeds = np.array(seeds)
    n = len(seeds)
    for pipelined in (False, True):
        tr = gnnv.Trainer(g, gnnv.Cache(g, 1.0), dims, fan, 4, w, prec=gnnv.PREC_TF32)
        try:
            assert tr.last_rows() and tr.fwd16()
            if pipelined:
                tr.prefetch(seeds, n, 41)
            loss, _ = tr.step(seeds, n, n, 41, 0.0)
            ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, fan, 41, w, 0.0)
            assert abs(loss - ref["loss"]) <= 5e-3 * abs(ref["loss"]), (pipelined, loss, ref["loss"])
            # every layer and dW/db through the oracle's chains over the
            # operands the GPU read (a 4-row batch leaves no averaging to
            # hide bf16 rounding in a normwise end-to-end bound)
            L = len(fan)
            hb = blocks_to_host(tr.blocks)
            grads = gnnv.unflat_params(tr.grads(), dims)
            X0 = oracle.gather_rows(gd.feats, hb[L - 1][4])[:, : dims[0]]
            tag = f"degenerate{n}{'p' if pipelined else 's'}"
            H, Aagg, blks = check_forward_chain(tr, hb, dims, w, RTOL[2], tag, X0=X0, max_rows=10**9)
            check_backward_chain(tr, blks, H, Aagg, dims, w, grads, gd.labels[seeds], n, RTOL[2], tag)
        finally:
            tr.free()


@pytest.mark.parametrize("kind", [gnnv.KIND_SAGE, gnnv.KIND_GCN])
@pytest.mark.parametrize("ratio", [0.3, 1.0])
def test_prefetched_layer1_aggregation_bitwise(mini, option, kind, ratio):
    """The Eq.4 prefetch also runs layer 1's aggregation (it needs no
    weight) for the batch it prepares, and the consuming step starts at the
    layer-1 GEMM (opt-in GNNV_PF_AGG; the default keeps it in the step): the same kernel on
    the same inputs, so three pipelined steps give bitwise the same losses,
    aggregates and activations (lr 0: the backward's atomic summation order
    would otherwise make the next weights differ at rounding level); ratio 1.0
    aggregates from the cache table, 0.3 from X."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    kname = "sage" if kind == gnnv.KIND_SAGE else "gcn"
    w = init_weights(dims, kind=kname)
    perm = epoch_seeds(gd.n, 0)
    out = {}
    for name in ("prefetch", "step"):
        option("GNNV_PF_AGG", 1 if name == "prefetch" else 0)
        tr = gnnv.Trainer(g, gnnv.Cache(g, ratio), dims, cfg["fanouts"], cfg["batch"], w, kind=kind,
                          prec=gnnv.PREC_FP32)
        res = []
        B = cfg["batch"]
        tr.prefetch(perm[:B], B, 60)
        for t in range(3):
            tr.step(perm[t * B:(t + 1) * B], B, B, 60 + t, 0.0, want_loss=False)
            if t < 2:
                tr.prefetch(perm[(t + 1) * B:(t + 2) * B], B, 61 + t)
            hb = blocks_to_host(tr.blocks)
            pa, sa = tr.aggregate(1)
            r = [tr.read_loss(), read_f32(pa, hb[L - 1][0], sa).tobytes()]
            for lvl in range(1, L + 1):
                p_, s_ = tr.activation(lvl)
                r.append(read_f32(p_, hb[L - lvl][0], s_).tobytes())
            res.append(r)
        out[name] = res
        tr.free()
    assert out["prefetch"] == out["step"]


@pytest.mark.parametrize("prec", [gnnv.PREC_FP32, gnnv.PREC_TF32])
@pytest.mark.parametrize("ratio", [0.3, 1.0])
def test_lastuse_l2_hints_bitwise_neutral(mini, option, prec, ratio):
    """The layer-1 aggregation's dead-row L2 hints (sampler: last-use slot
    per src id; evict_first on a row's last visit) change only cache
    priorities: the whole step -- loss, every activation level, the
    aggregates -- is bitwise identical with and without them
    (opt-in GNNV_LASTUSE); ratio 1.0 reads the cache table (rowidx), 0.3 reads X."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    out = {}
    for name in ("hints", "plain"):
        option("GNNV_LASTUSE", 1 if name == "hints" else 0)
        tr = gnnv.Trainer(g, gnnv.Cache(g, ratio), dims, cfg["fanouts"], cfg["batch"], w, prec=prec)
        loss, _ = tr.step(seeds, len(seeds), len(seeds), 0x5EED, 0.0)
        hb = blocks_to_host(tr.blocks)
        acts = [layer1_aggregate(tr, hb[L - 1][0])]
        for lvl in range(1, L):
            acts.append(read_activation(tr, lvl, hb[L - 1 - lvl][0]))
        out[name] = (loss, acts)
        tr.free()
    assert out["hints"][0] == out["plain"][0]
    for a_, b_ in zip(out["hints"][1], out["plain"][1]):
        assert a_.tobytes() == b_.tobytes()


@pytest.mark.parametrize("hidden", [64, 256])
def test_fwd16_resident_w_bitwise(mini, option, hidden):
    """Layer 1's bf16 forward GEMM with W^T resident in shared memory (the
    default when it fits) against the same GEMM streaming W^T with every A
    stage (GNNV_NO_BRES=1): the MMAs read the same operands in the same
    order, so the loss and every activation level (layer 1's bf16 copy, the
    later layers' rows) are bitwise identical; both forward epilogues store
    the ReLU bits after the proxy fence.  Hidden 64 and 256 (the resident
    image is BN x 128 bytes per k-block: 32 KB per k-block at 256)."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, hidden, hidden, gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    seeds = epoch_seeds(gd.n, 1)[: cfg["batch"]]
    out = {}
    for name in ("resident", "streamed"):
        option("GNNV_NO_BRES", 1 if name == "streamed" else 0)
        tr = gnnv.Trainer(g, gnnv.Cache(g, 1.0), dims, cfg["fanouts"], cfg["batch"], w, prec=gnnv.PREC_TF32)
        try:
            assert tr.fwd16()
            loss, _ = tr.step(seeds, len(seeds), len(seeds), 0xB2E5, 0.0)
            hb = blocks_to_host(tr.blocks)
            acts = [read_activation(tr, lvl, hb[L - 1 - lvl][0]) for lvl in range(1, L)]
            out[name] = (loss, acts)
        finally:
            tr.free()
    assert out["resident"][0] == out["streamed"][0]
    for a_, b_ in zip(out["resident"][1], out["streamed"][1]):
        assert a_.tobytes() == b_.tobytes()


@pytest.mark.parametrize("aggr", [gnnv.AGGR_MEAN, gnnv.AGGR_SUM])
@pytest.mark.parametrize("ratio", [0.3, 1.0])
def test_fused_l2_push_matches_per_layer_aggregation(mini, option, aggr, ratio):
    """The tf32 SAGE trainer (L >= 3) accumulates layer 2's aggregate in the
    layer-1 GEMM epilogue (L2 reductions over hop L-2's CSC) instead of
    storing H^1 and running the layer-2 aggregation; the default keeps the
    per-layer kernels.  Same step, same inputs: A^2 agrees to summation-order
    rounding, and the layer-2 output, the loss and the gradients to the tf32
    rounding that difference can move; ratio 1.0 also runs layer 1 from the
    cache table.  (Each path is checked against the oracle elsewhere:
    test_step_parity, test_gpu_fullsize.)"""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    out = {}
    for name in ("push", "plain"):
        option("GNNV_L2PUSH", 1 if name == "push" else 0)
        option("GNNV_NO_BF16ACT", 1)  # the push and the bf16 intermediates are exclusive
        tr = gnnv.Trainer(g, gnnv.Cache(g, ratio), dims, cfg["fanouts"], cfg["batch"], w, aggr=aggr,
                          prec=gnnv.PREC_TF32)
        assert tr.l2push() == (name == "push")
        tr.timeline(True)
        loss, _ = tr.step(seeds, len(seeds), len(seeds), 0x5EED, 0.05)
        segs = tr.timeline_read()
        hb = blocks_to_host(tr.blocks)
        pa, sa = tr.aggregate(2)
        p2, s2 = tr.activation(2)
        out[name] = dict(loss=loss, grads=tr.grads(), segs=segs, A2=read_f32(pa, hb[L - 2][0], sa)[:, : dims[1]],
                         H2=read_f32(p2, hb[L - 2][0], s2)[:, : dims[2]])
        tr.free()
    assert "spmm_fwd.l2" not in out["push"]["segs"] and "spmm_fwd.l2" in out["plain"]["segs"]
    p, q = out["push"], out["plain"]
    # A^2 differs only by summation order and w*x vs x/c rounding (~1 ulp);
    # downstream, an operand that lands on the other side of a tf32 rounding
    # boundary, or a pre-activation within that of zero, moves single
    # elements by up to 2^-10 of a term
    assert normwise(p["A2"], q["A2"]) < 1e-6
    assert normwise(p["H2"], q["H2"]) < 1e-4
    assert abs(p["loss"] - q["loss"]) <= 1e-5 * abs(q["loss"])
    assert normwise(p["grads"], q["grads"]) < 2e-3


@pytest.mark.parametrize("aggr", [gnnv.AGGR_MEAN, gnnv.AGGR_SUM])
def test_fused_output_layer_matches_per_kernel_path(mini, option, aggr):
    """The tf32 trainer runs its output layer (layer-L forward, CE loss,
    layer-L backward) as the two fused kernels of tail.cu; gnnv_set_option("GNNV_NO_TAIL", 1)
    (read when a trainer is created) keeps the seven per-kernel launches.
    Same step, same inputs: the loss, the logits, dH of layer L-1 and every
    gradient agree to the tf32 GEMM rounding, and both match the oracle."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    w = init_weights(dims)
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    out = {}
    for name in ("fused", "split"):
        option("GNNV_NO_TAIL", 1 if name == "split" else 0)
        tr = gnnv.Trainer(g, gnnv.Cache(g, cfg["ratio"]), dims, cfg["fanouts"], cfg["batch"], w, aggr=aggr,
                          prec=gnnv.PREC_TF32)
        tr.timeline(True)
        loss, _ = tr.step(seeds, len(seeds), len(seeds), 0x5EED, 0.05)
        segs = tr.timeline_read()
        hb = blocks_to_host(tr.blocks)
        pz, sz = tr.activation(L)
        pg, sg = tr.activation(L - 1)
        out[name] = dict(loss=loss, segs=segs, grads=tr.grads(), Z=read_f32(pz, hb[0][0], sz)[:, : gd.C])
    assert f"tail_a.l{L}" in out["fused"]["segs"] and "loss" not in out["fused"]["segs"]
    assert "loss" in out["split"]["segs"] and f"tail_a.l{L}" not in out["split"]["segs"]
    f, s = out["fused"], out["split"]
    assert abs(f["loss"] - s["loss"]) <= 2e-3 * abs(s["loss"])
    assert normwise(f["Z"], s["Z"]) < 4e-3
    assert normwise(f["grads"], s["grads"]) < 1e-2
    ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, cfg["fanouts"], 0x5EED, w, 0.05,
                     aggr="mean" if aggr == gnnv.AGGR_MEAN else "sum")
    assert abs(f["loss"] - ref["loss"]) <= 5e-3 * abs(ref["loss"])
    for (gW, gb), (rW, rb) in zip(gnnv.unflat_params(f["grads"], dims), ref["grads"]):
        for a_, b_ in ((gW, rW), (gb, rb)):
            cos = float(np.dot(a_.ravel(), b_.ravel()) / (np.linalg.norm(a_) * np.linalg.norm(b_) + 1e-30))
            assert cos > 0.98, cos


@pytest.mark.parametrize("d_in,d_out", [(100, 256), (64, 64), (64, 96)])
def test_layer_fwd_cta_pair_gemm(mini, option, d_in, d_out):
    """The CTA-pair (tcgen05 cta_group::2, M = 256) forward GEMM, GNNV_GEMM_PAIR=1:
    a tf32 SAGE layer forward equals the single-CTA GEMM's bit for bit (the
    same tf32 products accumulated in the same K order per output element)
    and the oracle within the tf32 bound -- with a ragged last pair (rows
    beyond n_dst in the peer CTA, never stored) and rows >= n_dst untouched."""
    gd, g = mini
    fan = CONFIGS["mini"]["fanouts"]
    seeds = epoch_seeds(gd.n, 0)[:300]
    blocks, hb = gpu_sample(g, seeds, fan, 11, max_seeds=512)
    layer, h = 2, 1
    ob = _oracle_block(hb, h)
    rng = np.random.default_rng(7)
    s_in = row_stride(d_in)
    Hsrc = np.zeros((ob.n_src, s_in), np.float32)
    Hsrc[:, :d_in] = rng.standard_normal((ob.n_src, d_in)).astype(np.float32)
    W = (rng.standard_normal((2 * d_in, d_out)) / np.sqrt(2 * d_in)).astype(np.float32)
    b = rng.standard_normal(d_out).astype(np.float32)
    ld = gnnv.layer_desc(d_in, d_out, s_in, 0, 0, 1, gnnv.PREC_TF32)
    view = blocks.info(sync=False)[h]
    cap_dst, cap_src = view.max_dst, view.max_src
    out = {}
    for pair in ("0", "1"):
        option("GNNV_GEMM_PAIR", int(pair))
        Hdst = torch.full((cap_dst, row_stride(d_out)), float("nan"), device="cuda")
        A = torch.full((cap_dst, s_in), float("nan"), device="cuda")
        gnnv.layer_fwd(blocks, layer, ld, padded(Hsrc, cap_src), dev_f32(W), dev_f32(b), Hdst, A)
        torch.cuda.synchronize()
        assert torch.isnan(Hdst[ob.n_dst:]).all()
        out[pair] = Hdst[: ob.n_dst].cpu().numpy()[:, :d_out]
    assert np.array_equal(out["0"], out["1"])
    Ho, _ = layer_fwd(ob, Hsrc[:, :d_in], W, b, True)
    Hm, _ = layer_fwd(ob, Hsrc[:, :d_in], W, b, True, absval=True)
    assert_close_cond(out["1"], Ho, Hm, RTOL[2], "pair GEMM layer")


@pytest.mark.parametrize("kind,prec", [(gnnv.KIND_SAGE, gnnv.PREC_FP32), (gnnv.KIND_GCN, gnnv.PREC_FP32),
                                       (gnnv.KIND_SAGE, gnnv.PREC_TF32)])
def test_backward_pull_matches_push(mini, option, kind, prec):
    """The backward aggregation of the layers with a dX (blocks h <= L-2)
    pulls per src row through the block's CSC (sampler: k_map counts, scan,
    k_csc_fill; k_spmm_bwd_pull) with GNNV_BWD_PULL=1 (read when the blocks
    handle is created); the default is the two-pass push (owner stores +
    atomic adds).
    Same step, same inputs: losses equal, gradients equal up to the
    summation order of repeated src ids (fp32) or the tf32 GEMM rounding,
    and both match the oracle's step (fp32: 1e-4 normwise)."""
    gd, g = mini
    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    kname = "sage" if kind == gnnv.KIND_SAGE else "gcn"
    w = init_weights(dims, kind=kname)
    seeds = epoch_seeds(gd.n, 0)[: cfg["batch"]]
    out = {}
    for name in ("push", "pull"):
        option("GNNV_BWD_PULL", 1 if name == "pull" else 0)
        tr = gnnv.Trainer(g, gnnv.Cache(g, cfg["ratio"]), dims, cfg["fanouts"], cfg["batch"], w, kind=kind,
                          prec=prec)
        tr.timeline(True)
        loss, _ = tr.step(seeds, len(seeds), len(seeds), 0x5EED, 0.05)
        out[name] = dict(loss=loss, grads=tr.grads(), segs=tr.timeline_read())
    p, q = out["pull"], out["push"]
    assert p["loss"] == q["loss"]  # the forward is untouched
    tol = 1e-5 if prec == gnnv.PREC_FP32 else 1e-2
    assert normwise(p["grads"], q["grads"]) < tol
    if prec == gnnv.PREC_FP32:
        ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, cfg["fanouts"], 0x5EED, w, 0.05,
                         kind=kname)
        for (gW, gb), (rW, rb) in zip(gnnv.unflat_params(p["grads"], dims, kind), ref["grads"]):
            assert normwise(gW, rW) < 1e-4 and normwise(gb, rb) < 1e-4


_GUARD_CHILD = r"""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.environ["GNNV_ROOT"], "tests"))
sys.path.insert(0, os.environ["GNNV_ROOT"])
import test_gpu_parity as t
t.lib()
from synth import make_graph
from paper_2404_09544_b200 import gnnv
gd = make_graph("mini")
t._guard_negative_control(gd, gnnv.Graph.from_data(gd))
print("GUARD_CHILD_OK")
"""


def test_guard_alloc_detects_out_of_bounds_write():
    """Negative control of the guarded-allocation check that stands in for
    compute-sanitizer (closed on this pool), in a child process with
    GNNV_GUARD_ALLOC=1: a kernel writing 12 floats past the end of a library
    allocation (gnnv_sgd over a range that ends beyond the trainer's H^1
    buffer) is reported; the guard is then restored."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GNNV_GUARD_ALLOC="1", GNNV_ROOT=root)
    r = subprocess.run([sys.executable, "-c", _GUARD_CHILD], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "GUARD_CHILD_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def _guard_negative_control(gd, g):
    import ctypes

    cfg = CONFIGS["mini"]
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    L = len(cfg["fanouts"])
    tr = gnnv.Trainer(g, gnnv.Cache(g, cfg["ratio"]), dims, cfg["fanouts"], cfg["batch"], init_weights(dims))
    tr.step(epoch_seeds(gd.n, 0)[: cfg["batch"]], cfg["batch"], cfg["batch"], 1, 0.0)
    assert gnnv.check_guards() == ""
    p1, s1 = tr.activation(1)
    rows = tr.blocks.info(sync=False)[L - 1].max_dst
    end = p1 + rows * s1 * 4
    ones = torch.ones(16, dtype=torch.float32, device="cuda")
    gnnv.sgd(end - 16, ones.data_ptr(), 16, -1.0)  # 4 floats inside, 12 past the end
    torch.cuda.synchronize()
    report = gnnv.check_guards()
    assert "H activations" in report and "after the end" in report, report
    rt = ctypes.CDLL("libcudart.so.12")
    assert rt.cudaMemset(ctypes.c_void_p(end), 0xA5, ctypes.c_size_t(48)) == 0
    torch.cuda.synchronize()
    assert gnnv.check_guards() == ""
    tr.free()
