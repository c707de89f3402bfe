python -c "import torch; print(torch.cuda.Stream.priority_range())"
for cfg in "-1 0" "0 0" "-1 -2" "-2 -1" "-1 -5" "-5 0"; do set -- $cfg
GNNV_STEP_PRIO=$1 GNNV_PF_PRIO=$2 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/prio.json 2>gpurun_out/prio.err || tail -3 gpurun_out/prio.err
python -c "import json; d=json.load(open('gpurun_out/prio.json')); print('step $1 pf $2', round(d['ms_per_step'],4), {k: round(v['avg_ms']*1000) for k,v in d['rooflines'].items()})"
done
