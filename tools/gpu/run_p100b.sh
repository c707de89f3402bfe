for v in 1 0; do
GNNV_HID16_DW=$v python bench.py --config papers100m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p100h_$v.json 2>gpurun_out/p100.err || tail -5 gpurun_out/p100.err
python -c "import json; d=json.load(open('gpurun_out/p100h_$v.json')); print('hid16dw=$v', round(d['value']), round(d['ms_per_step'],4), d['dtype'], {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items()})"
done
python -m pytest tests/test_gpu_parity.py -q -x -k "hidden" 2>&1 | tail -2
