python -c "import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)" 
for mb in 0 32 64 0 32 64; do
GNNV_L2WIN_MB=$mb timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/l2w_p_$mb.json 2>gpurun_out/l2w.err || tail -3 gpurun_out/l2w.err
GNNV_L2WIN_MB=$mb timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/l2w_s_$mb.json 2>>gpurun_out/l2w.err || tail -3 gpurun_out/l2w.err
python -c "import json; d=json.load(open('gpurun_out/l2w_p_$mb.json')); e=json.load(open('gpurun_out/l2w_s_$mb.json')); print($mb, round(d['ms_per_step'],4), round(e['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in e['rooflines'].items() if k in ('spmm_fwd.l1','gemm_fwd.l1','spmm_fwd.l2','gemm_dw.l1')})"
done
