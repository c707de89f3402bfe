#!/bin/bash
# One step's ncu --set full capture (serial step, products, tf32) and its
# launch list; writes gpurun_out/launches_np.csv, gpurun_out/ncu_step.ncu-rep.
set -e
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_np.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pipeline > /dev/null 2>&1
read SKIP COUNT < <(python - <<'PY'
import csv
lines=[l for l in open('gpurun_out/launches_np.csv') if l.startswith('"')]
names=[r['Kernel Name'] for r in csv.DictReader(lines) if r['Metric Name']=='gpu__time_duration.sum']
st=[i for i,n in enumerate(names) if 'k_init_seeds' in n]
print(st[3], st[4]-st[3])
PY
)
echo "skip $SKIP count $COUNT"
ncu --set full --clock-control none --import-source on --launch-skip $SKIP --launch-count $COUNT \
  -o gpurun_out/ncu_step -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/ncu_step.log 2>&1
