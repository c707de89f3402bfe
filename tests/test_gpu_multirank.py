"""-m gpu: the data-parallel GPU path at world size 2.

Two processes, one rank each (both on the box's one GPU), each run a whole
gnnv_step on its rank_slice of the global iteration with the loss scaled by
1/B_global (n_global = the global batch); the per-rank gradients and losses
are summed over a gloo process group on the host -- the exchange the NCCL
all-reduce performs on a multi-GPU box -- and the sum must equal the
oracle's single-process step on the concatenated batch (reading Q25,
Algorithm 1).  The ranks never wait on each other inside a kernel
(the sum happens on the host after each step), so this is not a stand-in
for a device collective.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, port: int, prec: int, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        from paper_2404_09544_b200 import gnnv
        from paper_2404_09544_b200.partition import global_batch, rank_slice
        from synth import BASE_RNG_SEED, CONFIGS, epoch_seeds, init_weights, make_graph

        torch.cuda.set_device(0)
        gnnv.load()
        cfg = CONFIGS["mini"]
        gd = make_graph("mini")
        g = gnnv.Graph.from_data(gd)
        cache = gnnv.Cache(g, cfg["ratio"])
        dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
        B = cfg["batch"] // 2  # per rank
        w = init_weights(dims)
        tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, w, prec=prec)
        perm = epoch_seeds(gd.n, 0)
        out = []
        for t in (0, 5):  # two global iterations; the second also exercises the Eq.4 prefetch
            lo, hi = rank_slice(t, rank, WORLD, B, gd.n)
            nglob = global_batch(t, WORLD, B, gd.n)
            if t == 5:
                tr.prefetch(perm[lo:hi], hi - lo, BASE_RNG_SEED + t)
            loss, _ = tr.step(perm[lo:hi], hi - lo, nglob, BASE_RNG_SEED + t, 0.0)
            g_loc = torch.as_tensor(np.concatenate([tr.grads(), [loss]]).astype(np.float64))
            dist.all_reduce(g_loc)  # the exchange step, on the host (gloo)
            out.append((t, g_loc.numpy()))
        tr.free()
        cache.free()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, "ERROR " + repr(e) + "\n" + traceback.format_exc()))


@pytest.mark.parametrize("prec", [0, 2], ids=["fp32", "tf32"])
def test_two_rank_gradient_sum_equals_concatenated_batch(prec):
    import torch.multiprocessing as mp

    from oracle.layers import train_step
    from paper_2404_09544_b200 import gnnv
    from paper_2404_09544_b200.partition import global_batch, rank_slice
    from synth import BASE_RNG_SEED, CONFIGS, epoch_seeds, init_weights, make_graph

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, prec, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(WORLD):
            r, res = q.get(timeout=300)
            results[r] = res
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(WORLD):
        assert not isinstance(results[r], str), results[r]
    cfg = CONFIGS["mini"]
    gd = make_graph("mini")
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    w = init_weights(dims)
    B = cfg["batch"] // 2
    perm = epoch_seeds(gd.n, 0)
    for k, (t, summed) in enumerate(results[0]):
        np.testing.assert_array_equal(summed, results[1][k][1])  # every rank holds the same sum
        lo0, _ = rank_slice(t, 0, WORLD, B, gd.n)
        seeds = perm[lo0:lo0 + global_batch(t, WORLD, B, gd.n)]  # the concatenated batch
        ref = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, cfg["fanouts"],
                         BASE_RNG_SEED + t, w, 0.0)
        got = gnnv.unflat_params(summed[:-1].astype(np.float32), dims)
        tol_loss, tol_g = (1e-5, 1e-4) if prec == 0 else (5e-3, None)
        assert abs(summed[-1] - ref["loss"]) <= tol_loss * abs(ref["loss"]), (t, summed[-1], ref["loss"])
        for i, ((gW, gb), (rW, rb)) in enumerate(zip(got, ref["grads"])):
            for a, b in ((gW, rW), (gb, rb)):
                if tol_g is not None:  # fp32: normwise, as the single-rank fp32 step test
                    err = float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
                    assert err <= tol_g, (t, i, err)
                else:  # tf32: the gradient direction (reading Q24)
                    cos = float(np.dot(a.ravel(), b.ravel()) / (np.linalg.norm(a) * np.linalg.norm(b) + 1e-30))
                    assert cos > 0.98, (t, i, cos)
