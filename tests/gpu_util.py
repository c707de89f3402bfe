"""Helpers for the -m gpu parity tests (CUDA path vs oracle)."""
import ctypes

import numpy as np
import torch

import oracle
from oracle.layers import agg_matrix, ce_loss, layer_bwd, layer_fwd
from oracle.sampler import Block

from paper_2404_09544_b200 import gnnv
from paper_2404_09544_b200.build import build

_built = False


def lib():
    global _built
    if not _built:
        build()
        _built = True
    return gnnv.load()


def dev_i32(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def dev_f32(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def read_i32(p, n):
    """Copy n int32 from a raw device pointer."""
    out = torch.empty(int(n), dtype=torch.int32, device="cuda")
    if n:
        torch.cuda.synchronize()
        res = _cudart().cudaMemcpy(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(int(p)),
                                   ctypes.c_size_t(int(n) * 4), 3)  # cudaMemcpyDeviceToDevice
        assert int(res) == 0, res
    return out.cpu().numpy()


def read_f32(p, rows, stride):
    """Copy a [rows x stride] fp32 matrix from a raw device pointer."""
    out = torch.empty((int(rows), int(stride)), dtype=torch.float32, device="cuda")
    if rows:
        torch.cuda.synchronize()
        res = _cudart().cudaMemcpy(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(int(p)),
                                   ctypes.c_size_t(int(rows) * int(stride) * 4), 3)
        assert int(res) == 0, res
    return out.cpu().numpy()


def read_bf16(p, rows, ld):
    """A [rows x ld] bf16 matrix from a device pointer, as float64."""
    n = int(rows) * int(ld)
    w = read_i32(p, (n + 1) // 2).view(np.uint16)[:n].reshape(int(rows), int(ld))
    return (w.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def bf16_round(x):
    """fp32 -> bf16 (round to nearest even, as __float2bfloat16_rn), as float64."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


def read_activation(tr, i, rows):
    """H^i's rows as stored: the fp32 rows, or -- when the trainer keeps none
    (H^1 at L = 3 with the bf16 hidden-layer paths) -- its bf16 copy."""
    p, s = tr.activation(i)
    if p:
        return read_f32(p, rows, s)
    p16, ld = tr.activation16(i)
    return read_bf16(p16, rows, ld)


def layer1_aggregate(tr, n_dst):
    """A^1 of the trainer's last step as stored: the fp32 rows, or -- when
    layer 1 keeps only the bf16 copy (gnnv_trainer_fwd16, reading Q33) --
    that copy (as float64)."""
    pa, sa = tr.aggregate(1)
    if pa:
        return read_f32(pa, n_dst, sa)
    _, p16, ld = tr.dw16_operands()
    return read_bf16(p16, n_dst, ld)


def read_bits(p, rows, words, ncols):
    """A [rows x words] uint32 ReLU bit mask from a device pointer, unpacked
    to bool [rows x ncols] (bit n%32 of word n/32)."""
    w = read_i32(p, int(rows) * int(words)).view(np.uint32).reshape(int(rows), int(words))
    bits = np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")
    return bits[:, :ncols].astype(bool)


_rt = None


def _cudart():
    global _rt
    if _rt is None:
        _rt = ctypes.CDLL("libcudart.so.12")
    return _rt


def blocks_to_host(blocks: gnnv.Blocks):
    """Per hop: (n_dst, n_src, indptr, indices, src_global) on the host.

    A trainer that leaves its last hop unrelabelled (gnnv_trainer_last_rows:
    indices are cache-table rows, F_L = F_{L-1}) is brought to the relabelled
    form here: rows -> vertex ids through the cache's degree order, then new
    local ids in first-appearance (CSR) order after F_{L-1} -- the numbering
    the sampler's scan gives -- so every check sees the same blocks."""
    torch.cuda.synchronize()
    views = blocks.info(sync=True)
    out = []
    for v in views:
        indptr = read_i32(v.d_indptr, v.n_dst + 1)
        indices = read_i32(v.d_indices, v.nnz)
        F = read_i32(v.d_src_global, v.n_src)
        out.append((int(v.n_dst), int(v.n_src), indptr, indices, F))
    order_ptr = getattr(blocks, "last_rows_order", None)
    if order_ptr:
        nd, ns, indptr, rows, F = out[-1]
        assert ns == nd, "last_rows: the last hop adds no frontier entries"
        order = read_i32(order_ptr, blocks.g.n)
        ids = order[rows]
        local = {int(u): i for i, u in enumerate(F)}
        Fl = list(F)
        idx = np.empty(len(ids), np.int32)
        for e, u in enumerate(ids.tolist()):
            j = local.get(u)
            if j is None:
                j = local[u] = len(Fl)
                Fl.append(u)
            idx[e] = j
        out[-1] = (nd, len(Fl), indptr, idx, np.asarray(Fl, np.int32))
    return out


def assert_close_cond(got, ref, mag, rtol, what=""):
    """Condition-aware elementwise bound (reading Q17):
    |got - ref| <= rtol * mag + 1e-30, mag = the same expression on |.|."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    mag = np.asarray(mag, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    err = np.abs(got - ref)
    bound = rtol * mag + 1e-30
    bad = err > bound
    if bad.any():
        i = np.unravel_index(np.argmax(err / bound), err.shape)
        raise AssertionError(f"{what}: {int(bad.sum())} of {err.size} elements exceed rtol={rtol}; worst at {i}: "
                             f"got {got[i]!r} ref {ref[i]!r} mag {mag[i]!r}")


def normwise(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def _blk(hb, h):
    nd, ns, ptr, idx, F = hb[h]
    return Block(n_dst=nd, n_src=ns, indptr=ptr.astype(np.int64), indices=idx.astype(np.int64), src_global=F)


def sub_block(ob: Block, H_src: np.ndarray, rows: np.ndarray):
    """The block restricted to dst rows `rows` (each output row depends only
    on its own sampled neighbours and itself): self rows first, then the
    neighbours' rows, so the oracle's layer_fwd applies unchanged."""
    cnt = np.diff(ob.indptr)[rows]
    nbr = np.concatenate([ob.indices[ob.indptr[r]:ob.indptr[r + 1]] for r in rows])
    n = len(rows)
    blk = Block(n_dst=n, n_src=n + nbr.size, indptr=np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64),
                indices=(n + np.arange(nbr.size)).astype(np.int64), src_global=None)
    return blk, np.concatenate([H_src[rows], H_src[nbr]])


def check_forward_chain(tr, hb, dims, w, rtol, name, X0=None, max_rows=2048, kind="sage", seed=0):
    """Every layer of the trainer's last forward against the oracle, each fed
    the GPU's own input (reading Q24); X0 = the exact layer-1 input when X
    is not materialised (whole-table cache).  Layers with more than max_rows
    output rows are checked on that many sampled rows (row-restricted
    blocks).  With the fused L2 push (tr.l2push()) layer i's GEMM also
    accumulated A^{i+1} and stored H^i for layer i+1's dst prefix only: layer
    i+1 is then checked on the GPU's [H^i_dst | A^{i+1}], and A^{i+1} itself
    against the aggregation of the oracle's layer i (from the GPU's input to
    layer i) on sampled rows, within layer i's bound (relu is 1-Lipschitz,
    the mean a convex sum).  Returns (H, Aagg, blks) for the backward."""
    L = len(hb)
    bf16 = tr.bf16act()
    push = tr.l2push() or bf16  # H^i stored in fp32 for the next dst prefix only
    rng = np.random.default_rng(seed)
    H = [None] * (L + 1)
    Aagg = [None] * (L + 1)
    blks = [None] * (L + 1)
    Hprev_in = None
    for i in range(1, L + 1):
        ob = blks[i] = _blk(hb, L - i)
        p_in, s_in = tr.activation(i - 1)
        p_out, s_out = tr.activation(i)
        # H^1 without fp32 rows (gnnv_trainer_activation NULL): its bf16 copy,
        # which is also what layer 2 read; the output check then allows the
        # copy's rounding on top of rtol
        out16 = not p_out and i >= 1
        in16 = not p_in and i >= 2
        pushed_in = push and 2 <= i <= L - 1  # A^i came from layer i-1's epilogue
        pushed_out = push and i <= L - 2  # H^i stored for the next dst prefix only
        if i == 1 and X0 is not None:
            Hin = X0
        elif pushed_in:
            Hin = read_activation(tr, i - 1, ob.n_dst)[:, : dims[i - 1]]  # the dst prefix the GPU stored
        else:
            Hin = read_activation(tr, i - 1, ob.n_src)[:, : dims[i - 1]]
        Hout = read_activation(tr, i, (_blk(hb, L - i - 1).n_dst if pushed_out else ob.n_dst))[:, : dims[i]]
        H[i - 1], H[i] = Hin, Hout
        Wi, bi = w[i - 1]
        if pushed_in and bf16:
            # layer i aggregated the bf16 copy of H^{i-1}: A^i against the
            # fp32 accumulation of exactly those bf16 values (1e-5), and the
            # copy against the fp32 prefix (bf16 rounding, 2^-9 relative)
            pa, sa = tr.aggregate(i)
            A_gpu = read_f32(pa, ob.n_dst, sa)[:, : dims[i - 1]]
            Aagg[i] = A_gpu
            p16, ld16 = tr.activation16(i - 1)
            H16 = read_bf16(p16, ob.n_src, ld16)[:, : dims[i - 1]]
            n_pre = len(Hin)
            np.testing.assert_allclose(H16[:n_pre], Hin, rtol=2.0 ** -8, atol=1e-30)
            A_ref = agg_matrix(ob, kind) @ H16
            A_mag = agg_matrix(ob, kind) @ np.abs(H16)
            assert_close_cond(A_gpu, A_ref, A_mag, 1e-5, f"{name} A^{i} over the bf16 copy of H^{i - 1}")
            X = np.concatenate([Hin.astype(np.float64), A_gpu.astype(np.float64)], axis=1)
            Z = X @ Wi.astype(np.float64) + bi
            Zm = np.abs(X) @ np.abs(Wi.astype(np.float64)) + np.abs(bi)
            Ho = np.maximum(Z, 0) if i < L else Z
            n = len(Hout)
            assert_close_cond(Hout, Ho[:n], Zm[:n], rtol, f"{name} layer {i} (on its bf16-fed aggregate)")
        elif pushed_in:
            pa, sa = tr.aggregate(i)
            A_gpu = read_f32(pa, ob.n_dst, sa)[:, : dims[i - 1]]
            Aagg[i] = A_gpu
            rows = np.sort(rng.choice(ob.n_dst, min(ob.n_dst, max_rows), replace=False))
            cnt = np.diff(ob.indptr)[rows]
            nbr = np.concatenate([ob.indices[ob.indptr[r]:ob.indptr[r + 1]] for r in rows])
            sub, Hs = sub_block(blks[i - 1], Hprev_in, nbr)
            Wp, bp = w[i - 2]
            Hn, _ = layer_fwd(sub, Hs, Wp, bp, True, kind)
            Hnm, _ = layer_fwd(sub, Hs, Wp, bp, True, kind, absval=True)
            seg = np.repeat(np.arange(len(rows)), cnt)
            wv = 1.0 / np.maximum(cnt, 1)
            A_ref = np.zeros((len(rows), dims[i - 1]))
            A_mag = np.zeros((len(rows), dims[i - 1]))
            np.add.at(A_ref, seg, Hn * wv[seg][:, None])
            np.add.at(A_mag, seg, Hnm * wv[seg][:, None])
            assert_close_cond(A_gpu[rows], A_ref, A_mag, rtol, f"{name} fused aggregate A^{i} (sampled rows)")
            X = np.concatenate([Hin.astype(np.float64), A_gpu.astype(np.float64)], axis=1)
            Z = X @ Wi.astype(np.float64) + bi
            Zm = np.abs(X) @ np.abs(Wi.astype(np.float64)) + np.abs(bi)
            Ho = np.maximum(Z, 0) if i < L else Z
            n = len(Hout)
            assert_close_cond(Hout, Ho[:n], Zm[:n], rtol, f"{name} layer {i} (on the fused aggregate)")
        elif len(Hout) > max_rows or pushed_out:  # only the stored prefix when pushed_out
            rows = np.sort(rng.choice(len(Hout), min(len(Hout), max_rows), replace=False))
            blk, Hs = sub_block(ob, Hin, rows)
            Ho, _ = layer_fwd(blk, Hs, Wi, bi, i < L, kind)
            Hm, _ = layer_fwd(blk, Hs, Wi, bi, i < L, kind, absval=True)
            if out16:  # the bf16 copy stands for the fp32 rows: + its rounding
                assert_close_cond(Hout[rows], Ho, (rtol + 2.0 ** -8) / rtol * Hm, rtol,
                                  f"{name} layer {i} (bf16 copy, sampled rows)")
            else:
                assert_close_cond(Hout[rows], Ho, Hm, rtol, f"{name} layer {i} (sampled rows)")
            if bf16 and pushed_out:  # the bf16 copy beyond the prefix, on sampled rows: + bf16 rounding
                p16, ld16 = tr.activation16(i)
                H16 = read_bf16(p16, ob.n_dst, ld16)[:, : dims[i]]
                rows = np.sort(rng.choice(ob.n_dst, min(ob.n_dst, max_rows), replace=False))
                blk, Hs = sub_block(ob, Hin, rows)
                Ho, _ = layer_fwd(blk, Hs, Wi, bi, i < L, kind)
                Hm, _ = layer_fwd(blk, Hs, Wi, bi, i < L, kind, absval=True)
                assert_close_cond(H16[rows], Ho, (rtol + 2.0 ** -8) / rtol * Hm, rtol,
                                  f"{name} bf16 copy of layer {i} (sampled rows)")
        else:
            Ho, _ = layer_fwd(ob, Hin, Wi, bi, i < L, kind)
            Hm, _ = layer_fwd(ob, Hin, Wi, bi, i < L, kind, absval=True)
            assert_close_cond(Hout, Ho, Hm, rtol, f"{name} layer {i}")
        Hprev_in = Hin
    return H, Aagg, blks


def check_backward_chain(tr, blks, H, Aagg, dims, w, grads, labels, n_global, rtol, name, kind="sage"):
    """Every dW/db elementwise against the oracle's backward chain run on the
    GPU's forward values (its logits, its ReLU masks): each GEMM stage
    between the loss and layer i adds at most rtol of the magnitude the same
    chain propagates on |.|.  With the fused push, layer i's ReLU mask comes
    from the GPU's bits and layer i+1's aggregate is the GPU's A^{i+1}."""
    L = len(blks) - 1
    push = tr.l2push() or tr.bf16act()
    _, G = ce_loss(H[L], labels, n_global)
    M = np.abs(G)
    for i in range(L, 0, -1):
        ob = blks[i]
        Hi = H[i]
        if push and i <= L - 2:  # H^i beyond the dst prefix exists only as its ReLU bits
            pbits, words = tr.relu_bits(i)
            Hi = read_bits(pbits, ob.n_dst, words, dims[i]).astype(np.float64)
        Hsrc = H[i - 1]
        if push and 2 <= i <= L - 1:
            A = Aagg[i].astype(np.float64)
            Hsrc = np.concatenate([H[i - 1], np.zeros((ob.n_src - ob.n_dst, dims[i - 1]), H[i - 1].dtype)])
        else:
            A = agg_matrix(ob, kind) @ H[i - 1].astype(np.float64)
        Wi = w[i - 1][0]
        rW, rb, rX = layer_bwd(ob, Hsrc, A, Hi, Wi, G, relu=(i < L), need_dx=(i > 1), kind=kind)
        mW, mb, mX = layer_bwd(ob, np.abs(Hsrc), np.abs(A), Hi, np.abs(Wi), M, relu=(i < L), need_dx=(i > 1),
                               kind=kind)
        stages = L - i + 1
        assert_close_cond(grads[i - 1][0], rW, mW, rtol * stages, f"{name} dW layer {i}")
        assert_close_cond(grads[i - 1][1], rb, mb, rtol * stages, f"{name} db layer {i}")
        G, M = rX, mX
