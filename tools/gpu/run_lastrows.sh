python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "bf16 or hidden or tiny or full_step or whole_table or prefetched or lastuse" 2>&1 | tail -3
for v in 0 1; do
GNNV_NO_LASTROWS=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/lr_$v.json 2>gpurun_out/lr.err || tail -5 gpurun_out/lr.err
GNNV_NO_LASTROWS=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/lr_serial_$v.json 2>>gpurun_out/lr.err
done
for f in gpurun_out/lr_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items()})"; done
