for v in 0 1 0 1; do
GNNV_PDL_PIPE=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/pdl_$v.json 2>gpurun_out/pdl.err || tail -5 gpurun_out/pdl.err
python -c "import json; d=json.load(open('gpurun_out/pdl_$v.json')); print('pdl $v', round(d['value']), round(d['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items()})"
done
