"""Ceiling argument for the layer-1 aggregation (spmm_fwd.l1) bytes.

The layer-1 aggregation reads, for every sampled edge of block b_{L-1}, one
400-byte feature row of the whole-table cache (products: ~2.46M edge visits
over ~1.35M distinct rows).  Its algorithmic bytes count each distinct row
once; DRAM sees a row again whenever it left L2 between two visits.  This
tool replays the kernel's row-visit sequence (dst rows in order, each row's
neighbours in CSR order -- the order the warps issue them) through an LRU
cache of the given capacities, with and without the aggregate's own output
rows allocating in L2, and reports misses / distinct rows: the DRAM re-read
factor no schedule in this order can beat with an L2 of that size (LRU is
near-optimal for this recency-free random pattern; Belady's bound is
reported too).  It also tries one reordering (dst rows sorted by the
smallest table row they read).

Runs on the GPU box (the blocks come from libgnnv's sampler on the bench's
batch) and prints one JSON line:
    python tools/l2_reuse_sim.py [--config products] [--t 10]
"""
import argparse
import json
import os
import sys
from collections import OrderedDict

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lru_misses(seq, cap_rows):
    d = OrderedDict()
    miss = 0
    for x in seq:
        if x in d:
            d.move_to_end(x)
        else:
            if x >= 0:
                miss += 1
            d[x] = None
            if len(d) > cap_rows:
                d.popitem(last=False)
    return miss


def belady_misses(seq, cap_rows):
    """Optimal offline replacement (evict the row whose next use is furthest)."""
    import heapq

    seq = np.asarray(seq)
    nxt = np.full(len(seq), len(seq), dtype=np.int64)
    last = {}
    for i in range(len(seq) - 1, -1, -1):
        x = int(seq[i])
        nxt[i] = last.get(x, len(seq))
        last[x] = i
    resident = {}
    heap = []
    miss = 0
    for i, x in enumerate(seq.tolist()):
        if x in resident:
            resident[x] = nxt[i]
            heapq.heappush(heap, (-nxt[i], x))
            continue
        miss += 1
        if len(resident) >= cap_rows:
            while True:
                nu, y = heapq.heappop(heap)
                if y in resident and resident[y] == -nu:
                    del resident[y]
                    break
        resident[x] = nxt[i]
        heapq.heappush(heap, (-nxt[i], x))
    return miss


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--t", type=int, default=10)
    a = ap.parse_args()
    import torch

    from paper_2404_09544_b200 import gnnv
    from synth import BASE_RNG_SEED, CONFIGS, epoch_seeds
    from synth.store import shared_graph

    gnnv.load()
    cfg = CONFIGS[a.config]
    gd = shared_graph(cfg)
    g = gnnv.Graph.from_data(gd)
    cache = gnnv.Cache(g, 1.0)
    B = cfg["batch"]
    seeds = epoch_seeds(gd.n, 0)[a.t * B:(a.t + 1) * B]
    blk = gnnv.Blocks(g, B, cfg["fanouts"])
    d = torch.as_tensor(seeds.astype(np.int32)).cuda()
    blk.sample(d.data_ptr(), B, BASE_RNG_SEED + a.t)
    views = blk.info(sync=True)
    L = len(cfg["fanouts"])
    v = views[L - 1]

    def rd(p, n):
        t = torch.empty(int(n), dtype=torch.int32, device="cuda")
        import ctypes

        ctypes.CDLL("libcudart.so.12").cudaMemcpy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(int(p)),
                                                  ctypes.c_size_t(int(n) * 4), 3)
        return t.cpu().numpy()

    indptr = rd(v.d_indptr, v.n_dst + 1)
    indices = rd(v.d_indices, v.nnz)
    FL = rd(v.d_src_global, v.n_src)
    slot = torch.empty(gd.n, dtype=torch.int32, device="cuda")
    import ctypes

    ctypes.CDLL("libcudart.so.12").cudaMemcpy(ctypes.c_void_p(slot.data_ptr()), ctypes.c_void_p(cache.info().d_slot),
                                              ctypes.c_size_t(gd.n * 4), 3)
    slot = slot.cpu().numpy()
    rows = slot[FL[indices]].astype(np.int64)  # table row of every edge visit, in issue order
    distinct = len(np.unique(rows))
    rowb = gd.stride * 4
    out = {"config": a.config, "edges": int(len(rows)), "distinct_rows": distinct, "row_bytes": rowb,
           "dst_rows": int(v.n_dst), "lru": {}, "lru_with_output_rows": {}, "belady": {}, "lru_minrow_order": {}}
    with_out = []
    ip = indptr.tolist()
    r = rows.tolist()
    for u in range(v.n_dst):
        with_out.extend(r[ip[u]:ip[u + 1]])
        with_out.append(-1 - u)  # the aggregate row written (allocates in L2)
    seg_min = np.full(v.n_dst, np.iinfo(np.int64).max)
    nz = np.diff(indptr) > 0
    seg_min[nz] = np.minimum.reduceat(rows, indptr[:-1][nz])
    order = np.argsort(seg_min, kind="stable")
    reord = np.concatenate([rows[indptr[u]:indptr[u + 1]] for u in order])
    for mb in (40, 63, 126):
        cap = int(mb * 1e6 / rowb)
        out["lru"][mb] = lru_misses(r, cap) / distinct
        out["lru_with_output_rows"][mb] = lru_misses(with_out, cap) / distinct
        out["lru_minrow_order"][mb] = lru_misses(reord.tolist(), cap) / distinct
        out["belady"][mb] = belady_misses(rows, cap) / distinct
    print(json.dumps(out))


if __name__ == "__main__":
    main()
