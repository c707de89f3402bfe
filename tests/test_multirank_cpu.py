"""The N>1 data-parallel path on CPU: world-size-2 gloo process groups.

Each rank takes its seed slice (paper_2404_09544_b200.partition), runs the
oracle iteration with the 1/B_global loss scale, and the gradients are
summed with all_reduce -- the same exchange the NCCL path performs.  The sum
must equal the single-process gradient of the concatenated batch
(reading Q25)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_09544_b200.partition import global_batch, iters_per_epoch, rank_slice


def test_rank_slices_cover_epoch_once():
    for n, world, batch in [(10, 1, 3), (10, 2, 3), (1000, 8, 37), (97, 3, 100), (2449029, 8, 4096)]:
        seen = np.zeros(n, dtype=np.int64)
        for t in range(iters_per_epoch(n, world, batch)):
            tot = 0
            for r in range(world):
                lo, hi = rank_slice(t, r, world, batch, n)
                assert 0 <= lo <= hi <= n and hi - lo <= batch
                seen[lo:hi] += 1
                tot += hi - lo
            assert tot == global_batch(t, world, batch, n)
        assert (seen == 1).all()
    assert iters_per_epoch(10, 1, 3) == 4  # |V|=10, |B0|=3 -> {3,3,3,1}
    assert [rank_slice(t, 0, 1, 3, 10)[1] - rank_slice(t, 0, 1, 3, 10)[0] for t in range(4)] == [3, 3, 3, 1]
    assert iters_per_epoch(1000, 1, 128) == 8
    with pytest.raises(ValueError):
        rank_slice(0, 2, 2, 3, 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.layers import train_step
        from synth import chung_lu_graph, epoch_seeds, init_weights, make_features, make_labels

        n, d, C = 3000, 8, 5
        indptr, indices = chung_lu_graph(n, 24000, 0.5, seed=7)
        feats, labels = make_features(n, d), make_labels(n, C)
        perm = epoch_seeds(n, 0)
        w = init_weights([d, 16, C])
        B, t = 40, 3
        lo, hi = rank_slice(t, rank, world, B, n)
        nglob = global_batch(t, world, B, n)
        out = train_step(indptr, indices, feats, d, labels, perm[lo:hi], [5, 4], 0x5EED + t, w, lr=0.0,
                         n_global=nglob)
        flat = np.concatenate([np.concatenate([g.ravel(), b.ravel()]) for g, b in out["grads"]] + [[out["loss"]]])
        buf = torch.tensor(flat, dtype=torch.float64)
        dist.all_reduce(buf)
        if rank == 0:
            glo, _ = rank_slice(t, 0, world, B, n)
            _, ghi = rank_slice(t, world - 1, world, B, n)
            full = train_step(indptr, indices, feats, d, labels, perm[glo:ghi], [5, 4], 0x5EED + t, w, lr=0.0)
            ref = np.concatenate([np.concatenate([g.ravel(), b.ravel()]) for g, b in full["grads"]] + [[full["loss"]]])
            q.put(float(np.abs(buf.numpy() - ref).max() / np.abs(ref).max()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_allreduced_grads_equal_concatenated_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    err = q.get(timeout=5)
    assert err < 1e-12, err
