set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "bf16_layer1_dw or bf16_intermediates or bf16_table" 2>&1 | tail -15
python -m pytest tests/test_gpu_fullsize.py -x -q -k products 2>&1 | tail -5
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/dw16_on_$i.json 2>gpurun_out/dw16_on.err
GNNV_NO_DW16=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/dw16_off_$i.json 2>>gpurun_out/dw16_on.err
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/dw16_on_serial.json 2>>gpurun_out/dw16_on.err
for f in gpurun_out/dw16_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d['ms_per_step'], d.get('roofline',{}).get('kernel'), d.get('phases_ms') or '')"; done
