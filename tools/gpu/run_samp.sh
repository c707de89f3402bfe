python -m pytest tests/test_gpu_parity.py -q -x -k "sample or relabel or hop or blocks" 2>&1 | tail -2
for v in 16384 131072; do
GNNV_GROUP_ROWS=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/samp_s_$v.json 2>gpurun_out/samp.err || tail -5 gpurun_out/samp.err
GNNV_GROUP_ROWS=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/samp_p_$v.json 2>>gpurun_out/samp.err
done
for f in gpurun_out/samp_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items() if 'sample' in k or 'gather' in k})"; done
