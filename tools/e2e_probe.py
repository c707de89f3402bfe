import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2404_09544_b200 import gnnv
from synth import BASE_RNG_SEED, CONFIGS, epoch_seeds, init_weights, make_graph
cfg = CONFIGS['products']; gd = make_graph(cfg); gnnv.load()
g = gnnv.Graph.from_data(gd); cache = gnnv.Cache(g, cfg['ratio'])
dims = [gd.d, 256, 256, gd.C]; B = cfg['batch']
tr = gnnv.Trainer(g, cache, dims, cfg['fanouts'], B, init_weights(dims), prec=gnnv.PREC_TF32)
perm = epoch_seeds(gd.n, 0).astype(np.int32); d_perm = torch.as_tensor(perm).cuda()
main = torch.cuda.Stream(priority=-1); torch.cuda.set_stream(main); pf = torch.cuda.Stream()
def loop(host, want_loss, steps=100, t0=10):
    S = lambda t: perm[t*B:(t+1)*B] if host else d_perm[t*B:(t+1)*B].data_ptr()
    tr.prefetch(S(t0), B, BASE_RNG_SEED+t0, on_host=host, stream=pf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main); prev=None; w0=time.perf_counter()
    for t in range(t0, t0+steps):
        tr.step(S(t), B, B, BASE_RNG_SEED+t, 0.01, on_host=host, want_loss=False, stream=main)
        tr.prefetch(S(t+1), B, BASE_RNG_SEED+t+1, on_host=host, stream=pf)
        if want_loss:
            tk = tr.loss_async(stream=main)
            if prev is not None: tr.loss_result(prev)
            prev = tk
    if want_loss: tr.loss_result(prev)
    e1.record(main); torch.cuda.synchronize(); wall=time.perf_counter()-w0
    tr.step(S(t0+steps), B, B, BASE_RNG_SEED+t0+steps, 0.01, on_host=host, want_loss=False, stream=main); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/steps, wall*1000/steps
for host in (False, True):
    for wl in (False, True):
        loop(host, wl, 20)
        print('host', host, 'loss', wl, ['%.3f' % x for x in loop(host, wl)])
