for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/spin_$i.json 2>gpurun_out/spin.err || tail -5 gpurun_out/spin.err
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/spin_serial.json 2>>gpurun_out/spin.err
for f in gpurun_out/spin_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items()})"; done
