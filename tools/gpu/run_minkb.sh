for kb in 1 8 16 24 32 48; do
GNNV_DW16_MINKB=$kb python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/minkb_$kb.json 2>gpurun_out/minkb.err || tail -3 gpurun_out/minkb.err
python -c "import json; d=json.load(open('gpurun_out/minkb_$kb.json')); print($kb, round(d['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items() if 'gemm_dw' in k})"
done
