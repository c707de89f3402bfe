for kb in 16 8 12 24 32 16; do
GNNV_DW16_MINKB=$kb python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/mk_p_$kb.json 2>gpurun_out/mk.err || tail -3 gpurun_out/mk.err
GNNV_DW16_MINKB=$kb python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/mk_s_$kb.json 2>>gpurun_out/mk.err
python -c "import json; d=json.load(open('gpurun_out/mk_p_$kb.json')); e=json.load(open('gpurun_out/mk_s_$kb.json')); print($kb, round(d['ms_per_step'],4), round(e['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in e['rooflines'].items() if 'gemm_dw' in k})"
done
