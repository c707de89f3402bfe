#!/bin/bash
# One bench line per BASELINE.json config (configs[0..4]; configs[2] at both
# ends of its cache sweep) -> gpurun_out/r02_bench_<config>@<ratio>.json (copied to profiles/)
mkdir -p gpurun_out profiles
for spec in "$@"; do
  IFS=: read CFG RATIO <<< "$spec"
  TAG="${CFG}@${RATIO}"
  echo "== $TAG"
  python bench.py --config "$CFG" --ratio "$RATIO" --steps 20 --warmup 5 > "gpurun_out/r02_bench_${TAG}.json" 2> "gpurun_out/bench_${TAG}.err" \
    || { echo "bench failed for $TAG"; tail -5 "gpurun_out/bench_${TAG}.err"; }
done
