python -m pytest tests/test_gpu_parity.py -x -q -k "bf16_layer1 or bf16_intermediates or bf16_table or full_step" 2>&1 | tail -15
python -m pytest tests/test_gpu_fullsize.py -x -q -k "products or papers" 2>&1 | tail -5
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/fwd16_on_$i.json 2>gpurun_out/fwd16.err
GNNV_NO_FWD16=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/fwd16_off_$i.json 2>>gpurun_out/fwd16.err
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/fwd16_on_serial.json 2>>gpurun_out/fwd16.err
for f in gpurun_out/fwd16_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1000) for k,v in d['phases_ms_per_step'].items()})"; done
