import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2404_09544_b200 import gnnv
from synth import CONFIGS, epoch_seeds, init_weights, make_graph, BASE_RNG_SEED
gnnv.load()
for name, B, fan, ratio in [("arxiv", 512, [15, 10, 5], 0.5), ("products", 4096, [15, 10, 5], 1.0)]:
    gd = make_graph(name); g = gnnv.Graph.from_data(gd)
    cfg = CONFIGS[name]; dims = [gd.d] + [cfg["hidden"]] * (len(fan) - 1) + [gd.C]
    cache = gnnv.Cache(g, ratio)
    tr = gnnv.Trainer(g, cache, dims, fan, B, init_weights(dims), prec=gnnv.PREC_TF32)
    perm = epoch_seeds(gd.n, 0); print('perm dtype', perm.dtype)
    d_perm = torch.as_tensor(perm).cuda(); nb = gd.n // B
    seeds = lambda t: d_perm[(t % nb) * B:((t % nb) + 1) * B].data_ptr()
    for t in range(3): tr.step(seeds(t), B, B, BASE_RNG_SEED + t, 0.01, on_host=False, want_loss=False)
    torch.cuda.synchronize()
    pf = torch.cuda.Stream(); main = torch.cuda.Stream(priority=-1)
    tr.prefetch(seeds(3), B, BASE_RNG_SEED + 3, on_host=False, stream=pf); torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(25)]
    evs[0].record(main)
    for i, t in enumerate(range(3, 27)):
        h0 = time.perf_counter()
        tr.step(seeds(t), B, B, BASE_RNG_SEED + t, 0.01, on_host=False, want_loss=False, stream=main)
        tr.prefetch(seeds(t + 1), B, BASE_RNG_SEED + t + 1, on_host=False, stream=pf)
        evs[i + 1].record(main)
        h1 = time.perf_counter()
        if h1 - h0 > 0.005: print('host call slow', i, round((h1 - h0) * 1e3, 2), 'ms')
    torch.cuda.synchronize()
    print(name, B, [round(evs[i].elapsed_time(evs[i + 1]), 3) for i in range(24)])
    tr.free(); cache.free()
