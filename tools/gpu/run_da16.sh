python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "bf16 or hidden or products or reddit or tf32 or pipelined or tail" 2>&1 | tail -3
for v in 0 1; do
GNNV_NO_DA16=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/da_$v.json 2>gpurun_out/da.err || tail -5 gpurun_out/da.err
GNNV_NO_DA16=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/da_serial_$v.json 2>>gpurun_out/da.err
done
python bench.py --config reddit --ratio 1.0 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/da_reddit.json 2>>gpurun_out/da.err
for f in gpurun_out/da_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items()})"; done
