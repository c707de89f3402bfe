python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_papers100m.py -q 2>&1 | tail -5
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/a16_on_$i.json 2>gpurun_out/a16.err || tail -5 gpurun_out/a16.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/a16_on_serial_$i.json 2>>gpurun_out/a16.err || { echo serial failed; grep -v CUDAEvent gpurun_out/a16.err | tail -5; }
done
for f in gpurun_out/a16_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), d['roofline']['kernel'], round(d['roofline']['frac'],3), {k: round(v*1000) for k,v in d['phases_ms_per_step'].items()})"; done
