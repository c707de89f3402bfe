"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into the
kernel sequence of one training step.

usage: python tools/launch_summary.py launches.csv [--step K] [--marker k_init_seeds]

Steps are delimited by launches of the marker kernel (the sampler's first
kernel); the K-th complete step is printed launch by launch with each
kernel's share of the step's summed kernel time.  ncu serialises launches
and runs them cold, so only the shares are comparable with bench.py.
"""
import argparse
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"^(void )?", "", name)
    name = name.split("(")[0]
    return name.replace("gnnv::", "")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--step", type=int, default=2)
    ap.add_argument("--marker", default="k_init_seeds")
    a = ap.parse_args()
    rows = []
    with open(a.csv) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        us = v / 1000.0 if unit == "ns" else (v if unit == "us" else v * 1000.0)
        rows.append((short(r["Kernel Name"]), r["Grid Size"], r["Block Size"], us))
    starts = [i for i, r in enumerate(rows) if r[0] == a.marker]
    if len(starts) < a.step + 2:
        sys.exit(f"only {len(starts)} steps in {a.csv}")
    seq = rows[starts[a.step]:starts[a.step + 1]]
    tot = sum(r[3] for r in seq)
    agg = defaultdict(float)
    print(f"step {a.step}: {len(seq)} launches, {tot:.1f} us summed kernel time (serialised, cold)")
    for name, grid, block, us in seq:
        agg[name] += us
        print(f"  {name:28s} grid {grid:>16s} block {block:>12s} {us:9.1f} us {100 * us / tot:5.1f}%")
    print("by kernel:")
    for name, us in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"  {name:28s} {us:9.1f} us {100 * us / tot:5.1f}%")


if __name__ == "__main__":
    main()
