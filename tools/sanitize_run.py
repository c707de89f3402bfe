"""Small end-to-end run of every libgnnv kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per gpurun call):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py

Covers: sampling (group- and thread-per-row, biased), relabel scan, gather
(HBM hits, zero-copy host misses, whole-table rowidx mode), SpMM forward and
the two-pass backward push, the tcgen05/TMA GEMMs (fwd, dX, dW) in tf32, the
bf16 and fp32 GEMMs, the fused output layer (tail), CE loss, SGD, the Eq.4
prefetch, the dynamic LRU cache admission.  Mini-sized (20K nodes).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_09544_b200 import gnnv  # noqa: E402
from synth import CONFIGS, epoch_seeds, init_weights, make_graph  # noqa: E402


def main():
    gnnv.load()
    torch.cuda.set_device(0)
    cfg = CONFIGS["mini"]
    gd = make_graph("mini")
    g = gnnv.Graph.from_data(gd)
    dims = [gd.d, cfg["hidden"], cfg["hidden"], gd.C]
    B = 256
    perm = epoch_seeds(gd.n, 0)
    done = []
    for ratio, prec in ((0.3, gnnv.PREC_TF32), (1.0, gnnv.PREC_TF32), (0.3, gnnv.PREC_BF16), (0.3, gnnv.PREC_FP32)):
        cache = gnnv.Cache(g, ratio)
        tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, init_weights(dims), prec=prec)
        tr.step(perm[:B], B, B, 1, 0.01)
        tr.prefetch(perm[B:2 * B], B, 2)  # Eq.4: side-stream sample + gather
        loss, _ = tr.step(perm[B:2 * B], B, B, 2, 0.01)
        assert np.isfinite(loss)
        done.append(f"ratio {ratio} prec {prec}: loss {loss:.4f}")
        tr.free()
        cache.free()
    # locality-biased sampler and the dynamic LRU cache
    cache = gnnv.Cache(g, 0.1, policy=gnnv.POLICY_LRU)
    tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, init_weights(dims), prec=gnnv.PREC_TF32)
    for t in range(3):
        tr.step(perm[t * B:(t + 1) * B], B, B, 10 + t, 0.01)
    tr.free()
    cache.free()
    cache = gnnv.Cache(g, 0.3)
    tr = gnnv.Trainer(g, cache, dims, [25, 10, 5], B, init_weights(dims), prec=gnnv.PREC_TF32)  # k > 16 sampler
    tr.set_locality(0.5)
    tr.step(perm[:B], B, B, 20, 0.01)
    tr.free()
    cache.free()
    torch.cuda.synchronize()
    print("sanitize_run ok:", "; ".join(done))


if __name__ == "__main__":
    main()
