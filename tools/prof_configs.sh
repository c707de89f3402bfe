#!/bin/bash
# Per-config ncu evidence (BASELINE.json configs[0..4]): one serial step's
# launches with their device time, DRAM bytes, PCIe bytes (the zero-copy
# host misses of Eq.6) and tensor-pipe activity, summarised per bench
# segment into gpurun_out/r02_ncu_traffic_<config>@<ratio>.json (copied to profiles/) (read back by
# bench.py's roofline `traffic`).  Each capture runs only after the same
# command exited 0 without ncu.
#   bash tools/prof_configs.sh cora:0.2:2 arxiv:0.5:3 reddit:0.1:2 reddit:1.0:2 products:1.0:3 papers100m:1.0:3
METRICS=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed
mkdir -p gpurun_out profiles
for spec in "$@"; do
  IFS=: read CFG RATIO L <<< "$spec"
  ARGS="--config $CFG --ratio $RATIO --steps 2 --warmup 3 --no-cpu-baseline --no-pipeline"
  TAG="${CFG}@${RATIO}"
  echo "== $TAG"
  if python bench.py $ARGS > "gpurun_out/plain_${TAG}.json" 2> "gpurun_out/plain_${TAG}.err"; then
    ncu --page raw --csv --metrics $METRICS --clock-control none --log-file "gpurun_out/ncu_${TAG}.csv" \
      python bench.py $ARGS > "gpurun_out/ncu_${TAG}.log" 2>&1
    python tools/ncu_traffic.py "gpurun_out/ncu_${TAG}.csv" --layers "$L" --workload "${CFG}@${RATIO}/tf32" --step 3 \
      --note "ncu --metrics (time, DRAM, PCIe, tensor pipe), one serial step (bench --no-pipeline, step 3 = first timed), cold caches per kernel replay" \
      > "gpurun_out/r02_ncu_traffic_${TAG}.json" || echo "summary failed for $TAG"
  else
    echo "plain run failed for $TAG"; tail -5 "gpurun_out/plain_${TAG}.err"
  fi
done
