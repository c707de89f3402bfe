#!/bin/bash
# A/B of library builds / env switches on the products workload, serial and
# pipelined.  Usage: VARIANTS="name:ENV=..;LIB=path ..." tools/ab_bench.sh
set -u
out=${OUT:-gpurun_out}
mkdir -p "$out"
for v in $VARIANTS; do
  name=${v%%:*}; envs=${v#*:}
  for mode in ${MODES:-serial pipe}; do
    extra=""; [ "$mode" = serial ] && extra="--no-pipeline"
    env $(echo "$envs" | tr ';' ' ') timeout 300 python bench.py --no-cpu-baseline --steps ${STEPS:-50} --warmup 10 $extra ${BENCH_ARGS:-} \
      > "$out/ab_${name}_${mode}.json" 2> "$out/ab_${name}_${mode}.err" || echo "fail $name $mode"
    python - "$out/ab_${name}_${mode}.json" "$name" "$mode" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[2], sys.argv[3], "no json", e); sys.exit(0)
r = d.get("rooflines", {})
def f(k):
    v = r.get(k); return f"{k} {v['avg_ms']*1e3:.0f}" if v else ""
print(sys.argv[2], sys.argv[3], f"{d['ms_per_step']:.3f} ms e2e {d.get('e2e',{}).get('value',0)/1e6:.3f}M", *[f(k) for k in ["spmm_fwd.l1","gather","pf_gather","gemm_fwd.l1","gemm_dw.l1","gemm_dw.l2","spmm_bwd.l2","pf_sample"]])
PY
  done
done
