"""-m gpu: the cross-GPU SHARDED cache placement (north_star: the feature
cache is sharded across the GPUs' HBM and read peer-to-peer).

Two ranks, one process each, exchange their shards' CUDA IPC handles over a
gloo process group (host-only gnnv comms), map each other's shard and
gather their own seed slice: rows bit-exact against the oracle and the
(rows, local hits, peer hits, host misses) counters equal to the oracle's
for that rank.  The box has one GPU, so both ranks map shards on the same
device through the same IPC path a multi-GPU box uses over NVLink; the
ranks never wait on each other inside a kernel (one-sided loads after a
host barrier), so this is not a stand-in for a collective.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WORLD = 2
RATIO = 0.6


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, port: int, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        import oracle
        from oracle.cache import access_counts, cache_slots
        from oracle.sampler import sample_blocks
        from paper_2404_09544_b200 import gnnv
        from paper_2404_09544_b200.partition import rank_slice
        from synth import CONFIGS, epoch_seeds, init_weights, make_graph

        torch.cuda.set_device(0)
        gnnv.load()
        cfg = CONFIGS["mini"]
        gd = make_graph("mini")
        g = gnnv.Graph.from_data(gd)
        comm = gnnv.Comm(rank, WORLD, None, 0)  # host-only: handles go over gloo
        cache = gnnv.Cache(g, RATIO, placement=gnnv.PLACE_SHARDED, comm=comm)
        B = cfg["batch"]
        lo, hi = rank_slice(0, rank, WORLD, B, gd.n)
        seeds = epoch_seeds(gd.n, 0)[lo:hi]
        blocks = gnnv.Blocks(g, len(seeds), cfg["fanouts"])
        d_seeds = torch.as_tensor(seeds.astype(np.int32)).cuda()
        blocks.sample(d_seeds.data_ptr(), len(seeds), 7)
        views = blocks.info()
        X = torch.empty((views[-1].max_src, gd.stride), dtype=torch.float32, device="cuda")
        stats = torch.zeros(4, dtype=torch.int64, device="cuda")
        state_err = False
        try:  # peers not mapped yet
            gnnv.gather(cache, blocks, X, stats)
        except gnnv.GnnvError as e:
            state_err = e.status == 2
        handles = [None] * WORLD
        dist.all_gather_object(handles, cache.ipc_handle())
        cache.open_peers(handles)
        dist.barrier()  # every shard filled and mapped
        gnnv.gather(cache, blocks, X, stats)
        torch.cuda.synchronize()
        F, _ = sample_blocks(gd.indptr, gd.indices, seeds, cfg["fanouts"], 7)
        FL = F[-1]
        rows_ok = X[: len(FL)].cpu().numpy().tobytes() == oracle.gather_rows(gd.feats, FL).tobytes()
        slot, owner, _ = cache_slots(gd.indptr, RATIO, world=WORLD)
        cnt = access_counts(slot, owner, FL, me=rank)
        want = [cnt["rows"], cnt["hits_local"], cnt["hits_peer"], cnt["misses_host"]]
        got = stats.cpu().tolist()
        # a whole training step through the trainer on the sharded cache
        dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
        tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], len(seeds), init_weights(dims), prec=gnnv.PREC_TF32)
        tr.step(seeds, len(seeds), len(seeds), 7, 0.01)
        p0, s0 = tr.activation(0)
        Xt = torch.empty((len(FL), s0), dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        import ctypes

        rt = ctypes.CDLL("libcudart.so.12")
        rt.cudaMemcpy(ctypes.c_void_p(Xt.data_ptr()), ctypes.c_void_p(p0), ctypes.c_size_t(Xt.numel() * 4), 3)
        step_ok = Xt.cpu().numpy().tobytes() == oracle.gather_rows(gd.feats, FL).tobytes()
        step_stats = tr.stats().tolist()
        dist.barrier()  # keep every shard alive until all ranks are done reading
        tr.free()
        cache.free()
        dist.destroy_process_group()
        q.put((rank, dict(state_err=state_err, rows_ok=rows_ok, got=got, want=want, step_ok=step_ok,
                          step_stats=step_stats)))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, "ERROR " + repr(e) + "\n" + traceback.format_exc()))


def test_sharded_cache_ipc_two_ranks():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(WORLD):
            r, res = q.get(timeout=240)
            results[r] = res
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(WORLD):
        res = results[r]
        assert isinstance(res, dict), res
        assert res["state_err"], "gather before open_peers must fail with STATE"
        assert res["rows_ok"], f"rank {r}: gathered rows differ from the oracle"
        assert res["got"] == res["want"], (r, res["got"], res["want"])
        assert res["want"][2] > 0, "the test must exercise peer reads"
        assert res["step_ok"] and res["step_stats"] == res["want"], (r, res)
