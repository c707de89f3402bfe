timeout 600 python -m pytest tests -m gpu -x -q -k "bf16 or tiny_batches or last_hop_table or full_step or resident_w" > gpurun_out/pt_epp.log 2>&1; tail -1 gpurun_out/pt_epp.log
for rep in 1 2; do
for v in on off; do
E=""; [ $v = off ] && E="GNNV_NO_EPPIPE=1"
env $E timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/epp_p_$v.json 2>gpurun_out/epp.err || tail -3 gpurun_out/epp.err
env $E timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/epp_s_$v.json 2>>gpurun_out/epp.err
python -c "import json; d=json.load(open('gpurun_out/epp_p_$v.json')); e=json.load(open('gpurun_out/epp_s_$v.json')); print('$v rep$rep', round(d['ms_per_step'],4), round(e['ms_per_step'],4), {k: round(v['avg_ms']*1000,1) for k,v in e['rooflines'].items() if 'gemm_fwd' in k})"
done
done
