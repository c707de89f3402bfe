python -m pytest tests/test_gpu_papers100m.py -q -x 2>&1 | tail -2
for v in 0 1; do
GNNV_NO_DW16=$v python bench.py --config papers100m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p100_$v.json 2>gpurun_out/p100.err || tail -5 gpurun_out/p100.err
python -c "import json; d=json.load(open('gpurun_out/p100_$v.json')); print('nodw16=$v', round(d['value']), round(d['ms_per_step'],4), d['dtype'], {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items()})"
done
