for cap in 0 148 296 74 444; do
GNNV_PF_CAP=$cap python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cap_$cap.json 2>gpurun_out/cap.err || tail -3 gpurun_out/cap.err
python -c "import json; d=json.load(open('gpurun_out/cap_$cap.json')); print($cap, round(d['value']), round(d['ms_per_step'],4), {k: round(v*1000) for k,v in d['phases_ms_per_step'].items()})"
done
