python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "bf16 or hidden or full_step or whole_table or lastuse or prefetched or stats or gather" 2>&1 | tail -3
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/rr_$i.json 2>gpurun_out/ri.err || tail -5 gpurun_out/ri.err
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/rr_serial.json 2>>gpurun_out/ri.err
python bench.py --config reddit --ratio 0.1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rr_reddit01.json 2>>gpurun_out/ri.err
for f in gpurun_out/rr_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['peaks'][-90:], {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items()})"; done
