"""Per-segment DRAM traffic of one training step from an `ncu --set full`
capture (raw page CSV), for bench.py's roofline `traffic` field.

usage:
  ncu --set full --clock-control none --launch-skip S --launch-count K -o step python bench.py --no-pipeline ...
  ncu -i step.ncu-rep --page raw --csv > step_raw.csv
  python tools/ncu_traffic.py step_raw.csv --layers 3 --workload products/tf32 > profiles/r01_ncu_traffic.json

The step's launches are assigned to the bench timeline's segments by the
trainer's fixed launch order (gnnv_step): sampler kernels -> "sample",
k_gather -> "gather", per layer k_spmm_fwd -> "spmm_fwd.l<i>", the forward
GEMM (+ its weight image) -> "gemm_fwd.l<i>", k_ce_loss -> "loss" (or the
fused output layer k_tail_a / k_tail_b -> "tail_a.l<L>" / "tail_b.l<L>"), per layer
from L down: mask pass -> "relu_mask.l<i>", dW GEMM + reductions ->
"gemm_dw.l<i>" (k_tma_dw16 too, with its bf16 G pass), dX GEMM (+ image) -> "gemm_dx.l<i>", the two aggregation
push passes -> "spmm_bwd.l<i>", k_sgd -> "sgd".  Traffic = dram__bytes_read
+ dram__bytes_write summed over the segment's kernels (ncu replays each
kernel with cold caches, so this is an upper bound on the in-step traffic).
"""
import argparse
import csv
import json
import re
import sys
from collections import OrderedDict

SAMPLER = ("k_init_seeds", "k_sample_hop", "k_winners", "k_relabel_scan", "k_map", "k_reset")


def short(name: str) -> str:
    name = re.sub(r"^(void )?", "", name).split("(")[0]
    name = re.sub(r"<\(int\)", "<", name)
    return name.replace("gnnv::", "").replace("tma::", "").replace("tc::", "")


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def to_us(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    return x * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1.0)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("raw_csv")
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--workload", default="products/tf32")
    ap.add_argument("--step", type=int, default=-1,
                    help="keep only the launches of the step-th gnnv_step (0-based; steps start at k_init_seeds)")
    ap.add_argument("--note", default="ncu --set full, one step (--no-pipeline), caches flushed per kernel replay")
    a = ap.parse_args()
    with open(a.raw_csv) as f:
        rows = [r for r in csv.reader(f)]
    h0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")  # skip ncu's log lines
    hdr, units, data = rows[h0], rows[h0 + 1], rows[h0 + 2:]
    ix = {h: i for i, h in enumerate(hdr)}
    launches = []
    for r in data:
        if len(r) < len(hdr):
            continue
        rd = to_bytes(r[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
        wr = to_bytes(r[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
        t = to_us(r[ix["gpu__time_duration.sum"]], units[ix["gpu__time_duration.sum"]])
        extra = {}
        for col, key in (("pcie__read_bytes.sum", "pcie_read"), ("pcie__write_bytes.sum", "pcie_write")):
            if col in ix and r[ix[col]] not in ("", "n/a"):
                extra[key] = to_bytes(r[ix[col]], units[ix[col]])
        col = "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"
        if col in ix and r[ix[col]] not in ("", "n/a"):
            extra["tensor_pct"] = float(r[ix[col]].replace(",", ""))
        launches.append((short(r[ix["Kernel Name"]]), rd, wr, t, extra))
    if a.step >= 0:  # the launches of one step: from its k_init_seeds to the next one
        starts = [i for i, k in enumerate(launches) if k[0].startswith("k_init_seeds")]
        lo = starts[a.step]
        hi = starts[a.step + 1] if a.step + 1 < len(starts) else len(launches)
        launches = launches[lo:hi]
    L = a.layers
    seg = OrderedDict()
    f, b, pending_dw, cur = 0, L + 1, False, None

    def add(name, k):
        s = seg.setdefault(name, {"dram_bytes": 0.0, "read": 0.0, "write": 0.0, "ncu_us": 0.0, "kernels": []})
        s["dram_bytes"] += k[1] + k[2]
        s["read"] += k[1]
        s["write"] += k[2]
        s["ncu_us"] += k[3]
        s["kernels"].append(k[0])
        for key in ("pcie_read", "pcie_write"):
            if key in k[4]:
                s[key] = s.get(key, 0.0) + k[4][key]
        if "tensor_pct" in k[4]:  # per kernel (a time-weighted figure is meaningless across kernels)
            s.setdefault("tensor_pipe_pct", []).append(round(k[4]["tensor_pct"], 2))

    for k in launches:
        n = k[0]
        if n.startswith(SAMPLER):
            cur = "sample"
        elif n.startswith("k_gather"):
            cur = "gather"
        elif n.startswith("k_spmm_fwd"):
            f += 1
            cur = f"spmm_fwd.l{f}"
        elif n.startswith(("k_bt_fwd", "k_wimg_fwd", "k_tma_gemm<0", "k_tc_gemm<0")):
            cur = f"gemm_fwd.l{f}"
        elif n.startswith("k_ce_loss"):
            cur = "loss"
        elif n.startswith("k_tail_a"):  # fused output layer (tail.cu): layer L fwd + loss + bwd
            cur = f"tail_a.l{f + 1}"
        elif n.startswith("k_tail_b"):
            cur = f"tail_b.l{L}"
            b = L
        elif n.startswith(("k_mask_colsum", "k_relu_mask", "k_relu_bits")):
            b -= 1
            pending_dw = True
            cur = f"relu_mask.l{b}"
        elif n.startswith("k_tma_dw16"):  # dW over bf16 operands
            if pending_dw:  # its G -> bf16 + db pass belongs to the same bench segment
                pending_dw = False
                m = seg.pop(f"relu_mask.l{b}", None)
                if m:
                    seg[f"gemm_dw.l{b}"] = m
            else:
                b -= 1
            cur = f"gemm_dw.l{b}"
        elif n.startswith(("k_tma_gemm<2", "k_tc_gemm<2", "k_gemm_simt")):
            if pending_dw:
                pending_dw = False
            else:
                b -= 1
            cur = f"gemm_dw.l{b}"
        elif n.startswith(("k_bt_dx", "k_wimg_dx", "k_tma_gemm<1", "k_tc_gemm<1")):
            cur = f"gemm_dx.l{b}"
        elif n.startswith("k_spmm_bwd"):
            cur = f"spmm_bwd.l{b}"
        elif n.startswith("k_sgd"):
            cur = "sgd"
        # reductions (k_dw_reduce*, k_colsum_reduce), k_zero_rows stay in the current segment
        if cur is None:
            sys.exit(f"unassigned launch {n}")
        add(cur, k)
    out = {"workload": a.workload, "source": a.raw_csv.split("/")[-1], "note": a.note, "segments": seg}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
