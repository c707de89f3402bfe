"""Summarise an `ncu --set full --import-source on` report of one kernel:
the launch's headline metrics and the source lines holding the most warp
stall samples (per file and line, first profiled kernel of the report).

    python tools/ncu_stall_summary.py gpurun_out/x.ncu-rep [--top 15]
"""
import argparse
import collections
import csv
import io
import subprocess

HEAD = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issued Warp Per Scheduler",
        "No Eligible", "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size",
        "Block Size", "L2 Hit Rate"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=15)
    ap.add_argument("--kernel", default="", help="substring of the kernel to summarise (default: the first)")
    a = ap.parse_args()
    filt = ["-k", f"regex:{a.kernel}", "-c", "1"] if a.kernel else []
    det = subprocess.run(["ncu", "-i", a.rep, "--page", "details", "--csv"] + filt, capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(det)))
    h = r[0]
    ki, ni, ui, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    seen = set()
    for x in r[1:]:
        if x[ii] != r[1][ii] or x[ni] not in HEAD or x[ni] in seen:
            continue
        seen.add(x[ni])
        print(f"{x[ki][:60]} | {x[ni]}: {x[vi]} {x[ui]}")
    src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + filt,
                         capture_output=True, text=True).stdout
    k, f = -1, None
    by, txt = collections.Counter(), {}
    for row in csv.reader(io.StringIO(src)):
        if row and row[0] == "Function Name":
            k += 1
            continue
        if row and row[0] == "File Path":
            f = row[1].split("/")[-1]
            continue
        if k != 0 or len(row) < 5 or not row[0].isdigit():
            continue
        try:
            v = float(row[4] or 0)
        except ValueError:
            continue
        by[(f, int(row[0]))] += v
        txt[(f, int(row[0]))] = row[1].strip()[:110]
    tot = sum(by.values()) or 1.0
    print(f"warp stall samples: {int(tot)}; top source lines (% of samples):")
    for key, v in by.most_common(a.top):
        print(f"  {key[0]}:{key[1]}  {100 * v / tot:5.1f}  {txt[key]}")


if __name__ == "__main__":
    main()
