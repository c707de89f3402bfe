python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "bf16 or products or whole_table or lastuse" 2>&1 | tail -3
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g16_$i.json 2>gpurun_out/g16.err || tail -5 gpurun_out/g16.err
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/g16_serial.json 2>>gpurun_out/g16.err
for f in gpurun_out/g16_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), d['roofline']['kernel'], round(d['roofline']['frac'],3), {k: round(v*1000) for k,v in d['phases_ms_per_step'].items()})"; done
