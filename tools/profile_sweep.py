"""Per-phase B200 profiles over a sweep of configurations, the training data
of the gray-box estimator (NEXT-4, paper_2404_09544_b200/estimator.py).

    python tools/profile_sweep.py OUT.jsonl [--quick]

Each record: the candidate (knobs + graph stats), measured frontier sizes
|F_h| and hit rate, per-phase times of the serial step (the library's
event timeline: sample, transfer = gather, replace = dynamic-cache
admission, compute = everything else), and the measured Eq.4-pipelined
step time for validating T.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_09544_b200 import gnnv  # noqa: E402
from synth import BASE_RNG_SEED, CONFIGS, epoch_seeds, init_weights, make_graph  # noqa: E402

SWEEP = [
    # graph, batch, fanouts, ratio, bias, policy
    ("arxiv", 512, [15, 10, 5], 0.5, 0.0, "degree"),
    ("arxiv", 1024, [15, 10, 5], 0.5, 0.0, "degree"),
    ("arxiv", 2048, [15, 10, 5], 1.0, 0.0, "degree"),
    ("arxiv", 1024, [10, 10], 0.2, 0.0, "degree"),
    ("arxiv", 1024, [15, 10, 5], 0.5, 1.0, "degree"),
    ("arxiv", 1024, [15, 10, 5], 0.2, 0.0, "lru"),
    ("products", 1024, [15, 10, 5], 1.0, 0.0, "degree"),
    ("products", 4096, [15, 10, 5], 1.0, 0.0, "degree"),
    ("products", 2048, [10, 5], 0.2, 0.0, "degree"),
    ("products", 4096, [15, 10, 5], 0.2, 0.0, "degree"),
    ("products", 2048, [15, 10, 5], 0.2, 1.0, "degree"),
    ("products", 2048, [15, 10, 5], 0.5, 0.0, "lru"),
    ("products", 4096, [10, 10, 10], 0.5, 0.0, "degree"),
    ("products", 2048, [20, 10], 1.0, 0.5, "degree"),
]
POLICY = {"degree": gnnv.POLICY_DEGREE, "fifo": gnnv.POLICY_FIFO, "lru": gnnv.POLICY_LRU}


def run(gd, g, name, B, fan, ratio, bias, policy, steps=12, warm=3):
    cfg = CONFIGS[name]
    dims = [gd.d] + [cfg["hidden"]] * (len(fan) - 1) + [gd.C]
    cache = gnnv.Cache(g, ratio, policy=POLICY[policy])
    tr = gnnv.Trainer(g, cache, dims, fan, B, init_weights(dims), prec=gnnv.PREC_TF32)
    tr.set_locality(bias)
    perm = epoch_seeds(gd.n, 0)
    d_perm = torch.as_tensor(perm).cuda()
    nb = gd.n // B

    def seeds(t):
        i = t % nb
        return d_perm[i * B:(i + 1) * B].data_ptr()

    for t in range(warm):
        tr.step(seeds(t), B, B, BASE_RNG_SEED + t, 0.01, on_host=False, want_loss=False)
    torch.cuda.synchronize()
    tr.timeline(True)
    frontier = np.zeros(len(fan) + 1)
    hits = rows = 0
    for t in range(warm, warm + steps):
        tr.step(seeds(t), B, B, BASE_RNG_SEED + t, 0.01, on_host=False, want_loss=False)
        views = tr.blocks.info(sync=True)
        frontier += np.array([views[0].n_dst] + [v.n_src for v in views])
        st = tr.stats()
        rows += int(st[0])
        hits += int(st[1] + st[2])
    segs = tr.timeline_read()
    tr.timeline(False)
    ph = {"sample": 0.0, "transfer": 0.0, "replace": 0.0, "compute": 0.0}
    for k, (ms, _) in segs.items():
        if k == "sample":
            ph["sample"] += ms
        elif k == "gather":
            ph["transfer"] += ms
        elif k == "replace":
            ph["replace"] += ms
        else:
            ph["compute"] += ms
    ph = {k: v / steps for k, v in ph.items()}
    # Eq.4 pipelined step time (device clock)
    pf = torch.cuda.Stream()
    main = torch.cuda.Stream(priority=-1)  # as bench.py: non-default, high priority
    t0 = warm + steps
    tr.prefetch(seeds(t0), B, BASE_RNG_SEED + t0, on_host=False, stream=pf)
    for t in range(t0, t0 + 2):  # untimed pipelined warm-up (both buffer sets in use)
        tr.step(seeds(t), B, B, BASE_RNG_SEED + t, 0.01, on_host=False, want_loss=False, stream=main)
        tr.prefetch(seeds(t + 1), B, BASE_RNG_SEED + t + 1, on_host=False, stream=pf)
    t0 += 2
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for t in range(t0, t0 + steps):
        tr.step(seeds(t), B, B, BASE_RNG_SEED + t, 0.01, on_host=False, want_loss=False, stream=main)
        tr.prefetch(seeds(t + 1), B, BASE_RNG_SEED + t + 1, on_host=False, stream=pf)
    e1.record(main)
    torch.cuda.synchronize()
    pipe_ms = e0.elapsed_time(e1) / steps
    tr.step(seeds(t0 + steps), B, B, BASE_RNG_SEED + t0 + steps, 0.01, on_host=False, want_loss=False,
            stream=main)
    torch.cuda.synchronize()
    tr.free()
    cache.free()
    cand = dict(n_nodes=gd.n, nnz=gd.nnz, n_attr=gd.d, stride=gd.stride, n_classes=gd.C, batch=B, fanouts=fan,
                hidden=cfg["hidden"], ratio=ratio, locality_bias=bias, policy=policy, kind="sage")
    return dict(graph=name, candidate=cand, frontier=(frontier / steps).tolist(), hit=hits / max(1, rows),
                phases_ms=ph, serial_ms=sum(ph.values()), pipelined_ms=pipe_ms)


def main():
    out = sys.argv[1]
    quick = "--quick" in sys.argv
    gnnv.load()
    graphs = {}
    with open(out, "w") as f:
        for (name, B, fan, ratio, bias, policy) in (SWEEP[:3] if quick else SWEEP):
            if name not in graphs:
                t = time.time()
                gd = make_graph(name)
                graphs[name] = (gd, gnnv.Graph.from_data(gd))
                print(f"graph {name}: {time.time() - t:.1f} s", file=sys.stderr)
            gd, g = graphs[name]
            rec = run(gd, g, name, B, fan, ratio, bias, policy)
            print(json.dumps(rec), file=f, flush=True)
            print(name, B, fan, ratio, bias, policy, {k: round(v, 3) for k, v in rec["phases_ms"].items()},
                  round(rec["pipelined_ms"], 3), file=sys.stderr)


if __name__ == "__main__":
    main()
