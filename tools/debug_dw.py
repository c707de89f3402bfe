"""Debug helper: one tf32 dW (GCN, single source) through gnnv_layer_bwd on a
small sampled block, compared with numpy.  Build with GNNV_DEBUG_DW to get
kernel printf output."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2404_09544_b200 import gnnv
from synth import make_graph, epoch_seeds, row_stride
from oracle.layers import layer_bwd
from oracle.sampler import Block
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from gpu_util import blocks_to_host, dev_f32, dev_i32

gd = make_graph("mini")
g = gnnv.Graph.from_data(gd)
d_in, d_out = int(sys.argv[1]) if len(sys.argv) > 1 else 32, int(sys.argv[2]) if len(sys.argv) > 2 else 32
blocks = gnnv.Blocks(g, 64, [5])
seeds = epoch_seeds(gd.n, 0)[:64]
blocks.sample(dev_i32(seeds), 64, 1)
hb = blocks_to_host(blocks)
nd, ns, ptr, idx, F = hb[0]
ob = Block(nd, ns, ptr.astype(np.int64), idx.astype(np.int64), F)
rng = np.random.default_rng(0)
s_in = row_stride(d_in)
H = np.zeros((ns, s_in), np.float32); H[:, :d_in] = 1 + rng.integers(0, 3, (ns, d_in))
A = np.zeros((nd, s_in), np.float32); A[:, :d_in] = H[:nd, :d_in]
W = np.ones((d_in, d_out), np.float32)
so = row_stride(d_out)
G = np.zeros((nd, so), np.float32); G[:, :d_out] = 1
Hd = np.ones((nd, so), np.float32)
dW = torch.zeros((d_in, d_out), device="cuda"); db = torch.zeros(d_out, device="cuda")
ld = gnnv.layer_desc(d_in, d_out, s_in, gnnv.KIND_GCN, 0, 0, 2)
gnnv.layer_bwd(blocks, 1, ld, dev_f32(G), dev_f32(Hd), dev_f32(H), dev_f32(A), dev_f32(W), None, dW, db)
torch.cuda.synchronize()
ref = A[:, :d_in].astype(np.float64).T @ G[:, :d_out]
got = dW.cpu().numpy()
print("nd", nd, "got[0,:4]", got[0, :4], "ref[0,:4]", ref[0, :4], "maxerr", np.abs(got - ref).max())
print("db", db.cpu().numpy()[:4], "ref", G[:, :d_out].sum(0)[:4])
