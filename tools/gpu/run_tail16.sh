python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "bf16 or hidden or products or tf32 or pipelined or tail" 2>&1 | tail -3
for v in 0 1; do
GNNV_NO_TAIL16=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/t16_$v.json 2>gpurun_out/t16.err || tail -5 gpurun_out/t16.err
GNNV_NO_TAIL16=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/t16_serial_$v.json 2>>gpurun_out/t16.err
done
for f in gpurun_out/t16_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items()})"; done
