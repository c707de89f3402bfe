"""Micro-benchmark of the dense layer products at the products-config shapes.

    python tools/bench_gemm.py [M] [d_in] [d_out]
Prints device time and achieved HBM GB/s of the tf32 TMA kernels (the
round-1 switches that disabled the epilogue stores / the MMA were removed
from the product kernel).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09544_b200 import gnnv  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 492000
d_in = int(sys.argv[2]) if len(sys.argv) > 2 else 100
d_out = int(sys.argv[3]) if len(sys.argv) > 3 else 256
ld_in, ld_out = (d_in + 3) & ~3, (d_out + 3) & ~3
g = torch.Generator(device="cuda").manual_seed(0)
X1 = torch.randn(M, ld_in, device="cuda", generator=g)
X2 = torch.randn(M, ld_in, device="cuda", generator=g)
W = torch.randn(2 * d_in, d_out, device="cuda", generator=g) * 0.05
b = torch.randn(d_out, device="cuda", generator=g)
Y = torch.empty(M, ld_out, device="cuda")
G = torch.randn(M, ld_out, device="cuda", generator=g)
dW = torch.empty(2 * d_in, d_out, device="cuda")
db = torch.empty(d_out, device="cuda")
Y1 = torch.empty(M, ld_in, device="cuda")
Y2 = torch.empty(M, ld_in, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for prec, pname in [(gnnv.PREC_TF32, "tf32"), (gnnv.PREC_FP32, "fp32")]:
    t_fwd = timeit(lambda: gnnv.dense_fwd(X1, ld_in, X2, ld_in, d_in, W, b, Y, ld_out, d_out, M, True, prec))
    by = M * 2 * d_in * 4 + M * ld_out * 4
    print(f"{pname} fwd  M={M} K={2*d_in} N={d_out}: {t_fwd*1e3:8.1f} us  {by/t_fwd/1e6:7.0f} GB/s")
    t_dx = timeit(lambda: gnnv.dense_dx(G, ld_out, d_out, W, d_in, Y1, ld_in, Y2, ld_in, M, prec))
    by = M * d_out * 4 + M * 2 * ld_in * 4
    print(f"{pname} dx   : {t_dx*1e3:8.1f} us  {by/t_dx/1e6:7.0f} GB/s")
    t_dw = timeit(lambda: gnnv.dense_dw(X1, ld_in, X2, ld_in, d_in, G, ld_out, d_out, M, dW, db, prec))
    by = M * 2 * d_in * 4 + M * d_out * 4
    print(f"{pname} dw   : {t_dw*1e3:8.1f} us  {by/t_dw/1e6:7.0f} GB/s  (incl. db colsum for tf32)")
