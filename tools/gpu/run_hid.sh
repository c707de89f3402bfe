python -m pytest tests/test_gpu_parity.py -q -x -k "bf16 or hidden or full_step or tf32" 2>&1 | tail -4
python -m pytest tests/test_gpu_fullsize.py -q -x -k "products or arxiv" 2>&1 | tail -3
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/hid_$i.json 2>gpurun_out/hid.err || tail -5 gpurun_out/hid.err
done
GNNV_NO_HID16=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/hid_off.json 2>>gpurun_out/hid.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/hid_serial.json 2>>gpurun_out/hid.err
for f in gpurun_out/hid_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), d['roofline']['kernel'], round(d['roofline']['frac'],3), {k: (round(v['avg_ms']*1000), round(v['frac'],2)) for k,v in d['rooflines'].items()})"; done
