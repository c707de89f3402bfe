python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "bf16 or hidden or tiny or full_step or whole_table or prefetched or lastuse or step" 2>&1 | tail -3
for rep in 1 2; do
for v in 0 1; do
GNNV_KEEP_H1=$v python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/h1_$v.json 2>gpurun_out/h1.err || tail -5 gpurun_out/h1.err
python -c "import json; d=json.load(open('gpurun_out/h1_$v.json')); print('keep_h1=$v rep$rep', round(d['value']), round(d['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items() if k in ('gemm_fwd.l1','pf_sample','spmm_fwd.l1')})"
done
done
