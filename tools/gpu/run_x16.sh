python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "bf16 or hidden or whole_table or lastuse or products or prefetched" 2>&1 | tail -3
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/x16_$i.json 2>gpurun_out/x16.err || tail -5 gpurun_out/x16.err
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/x16_serial.json 2>>gpurun_out/x16.err
for f in gpurun_out/x16_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), {k: (round(v['avg_ms']*1000), round(v['frac'],2)) for k,v in d['rooflines'].items()})"; done
