#!/usr/bin/env python
"""Benchmark: sampled-GraphSAGE training iterations (GNNavigator hot path) on B200.

One step = one whole iteration of Algorithm 1 per rank:
sample -> gather (degree cache) -> 3 x (SpMM aggregate + dense transform) ->
softmax-CE loss -> backward -> NCCL all-reduce -> SGD, through the libgnnv
C-ABI (gnnv_step).  Workload: the ogbn-products-shaped synthetic graph
(BASELINE.json configs[3]: 2.45M nodes, 61.9M CSR edges, d=100, 47 classes,
fanouts [15,10,5], 4096 seeds per rank, cache ratio 1.0 replicated).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0 (see DESIGN.md §6 for every field).
`--impl reference` times the CPU oracle (oracle/) on the same workload: the
paper ships no code, so the oracle is this tier's reference arm.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "sampled-GraphSAGE seeds/sec"
UNIT = "seeds/s"
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 148 SMs x 128 FP32 lanes x FMA x 1.965 GHz (guide)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="products")
    p.add_argument("--prec", default="tf32", choices=["fp32", "bf16", "tf32"])
    p.add_argument("--kind", default="sage", choices=["sage", "gcn"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-baseline-seeds", type=int, default=0, help="seeds in the oracle sample (0 = one batch)")
    p.add_argument("--ratio", type=float, default=None)
    p.add_argument("--policy", default="degree", choices=["degree", "fifo", "lru", "none"],
                   help="cache policy: static degree template, or dynamic FIFO/LRU admission (NEXT-3)")
    p.add_argument("--locality-bias", type=float, default=0.0,
                   help="NEXT-2 locality-biased sampling: cached neighbours weigh 1 + 4*bias (bias in 0, .25, .5, .75, 1)")
    p.add_argument("--placement", default="replica", choices=["replica", "sharded"],
                   help="feature cache across ranks: replicated, or sharded over the GPUs' HBM (NVLink peer reads)")
    p.add_argument("--no-pipeline", action="store_true",
                   help="disable the Eq.4 overlap of next-batch sample+gather with compute")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        pk = json.load(open(path))
        return dict(hbm=float(pk["hbm_gbs"]), bf16=float(pk["bf16_tflops"]),
                    bf16_sust=float(pk["bf16_tflops_sustained"]), src="measured (MEASURED_PEAKS.json)")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sust=1400.0, src="fallback (B200_PROFILING.md)")


def measure_host_link() -> float:
    """Host->device bandwidth of this box (GB/s), the roofline of the cache
    misses' zero-copy reads (Eq.6): the better of the copy engine (best of 5
    pinned 256 MB copies) and SM zero-copy reads of the same pinned buffer
    (gnnv_host_read_probe: the gather's own access pattern, 16-byte loads
    from every SM), each the best of 5."""
    import torch

    from paper_2404_09544_b200 import gnnv

    src = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    dst = torch.empty_like(src, device="cuda")
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, src.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9)
    try:
        for _ in range(5):
            ms = gnnv.host_read_probe(src.data_ptr(), src.numel(), 1)
            best = max(best, src.numel() / (ms / 1e3) / 1e9)
    except Exception:
        pass
    return best


def load_traffic(workload: str):
    """Per-segment DRAM bytes of one step from the committed ncu captures
    (tools/ncu_traffic.py -> profiles/r*_ncu_traffic*.json, newest round
    first) for this workload ("<config>/<prec>"), or {}."""
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_traffic*.json")), reverse=True):
        try:
            d = json.load(open(path))
            if d.get("workload") == workload:
                return {k: v["dram_bytes"] for k, v in d["segments"].items()}
        except Exception:
            pass
    return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=1)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "reasons": sorted(reasons), "samples": len(sm)}


def d2d(dst, src_ptr: int, nbytes: int):
    """Device-to-device copy from a raw libgnnv pointer into a torch tensor."""
    import ctypes

    rt = ctypes.CDLL("libcudart.so.12")
    rc = rt.cudaMemcpy(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(int(src_ptr)), ctypes.c_size_t(nbytes), 3)
    if rc != 0:
        raise RuntimeError(f"cudaMemcpy failed: {rc}")


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform

    return platform.processor() or "unknown"


# ---------------------------------------------------------------- oracle arm
# P = len(sched_getaffinity) worker processes, BLAS threads 1
# each, every worker maps the shared host store (/dev/shm, synth.store) and
# runs the oracle's train_step (oracle/layers.py, as it stands) on its own
# contiguous slice of the global batch -- as ranks would; the main process
# sums the slices' gradients (the all-reduce) and applies the oracle's SGD.
_WORKER = {}


def _oracle_init(store_path):
    from threadpoolctl import threadpool_limits

    _WORKER["limits"] = threadpool_limits(1)  # one BLAS/OpenMP thread per worker process
    from synth.store import open_store

    _WORKER["gd"] = open_store(store_path)


def _oracle_slice(job):
    from oracle.layers import train_step

    seeds, rs, weights, n_global, fanouts, kind = job
    gd = _WORKER["gd"]
    out = train_step(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, seeds, fanouts, rs, weights, 0.0,
                     n_global=n_global, kind=kind)
    return out["loss"], out["grads"]


class OracleArm:
    """The CPU oracle over `procs` worker processes (spawned, so none of them
    inherits a CUDA context)."""

    def __init__(self, gd, cfg, kind, procs):
        import multiprocessing as mp

        from synth.store import store_path, write_store

        self.cfg, self.kind, self.procs = cfg, kind, procs
        path = store_path(cfg)
        if not os.path.isdir(path):  # bench ranks normally created it already
            write_store(gd, cfg)
        self.pool = mp.get_context("spawn").Pool(procs, initializer=_oracle_init, initargs=(path,))

    def step(self, seeds, rs, weights, lr):
        """One oracle iteration on the global batch `seeds`; returns new weights."""
        from oracle.layers import sgd_update

        P = min(self.procs, len(seeds))
        cuts = np.linspace(0, len(seeds), P + 1).astype(int)
        jobs = [(seeds[cuts[i]:cuts[i + 1]], rs, weights, len(seeds), self.cfg["fanouts"], self.kind) for i in range(P)]
        outs = self.pool.map(_oracle_slice, jobs)
        grads = [[sum(o[1][l][j] for o in outs) for j in range(2)] for l in range(len(weights))]
        return [tuple(sgd_update([W, b], g, lr)) for (W, b), g in zip(weights, grads)]

    def time(self, seeds_list, rs_list, weights, lr):
        t0 = time.perf_counter()
        n = 0
        for seeds, rs in zip(seeds_list, rs_list):
            weights = self.step(seeds, rs, weights, lr)
            n += len(seeds)
        return n, time.perf_counter() - t0, weights

    def close(self):
        self.pool.close()
        self.pool.join()


def oracle_baseline(gd, cfg, kind, perm, seeds_of_t, t0, weights, lr, budget_s=20.0):
    """cpu_baseline: the oracle on the same workload, host cores of this box:
    full global batches with P workers until ~budget_s, plus a 1-core figure
    (one worker process, one BLAS thread) on one rank-sized slice of B/P."""
    P = cpu_cores()
    arm = OracleArm(gd, cfg, kind, P)
    try:
        arm.time([seeds_of_t(t0)[: 16 * P]], [BASE_RNG_SEED_BENCH - 1], weights, lr)  # worker start-up, untimed
        n, tt, its = 0, 0.0, 0
        w = weights
        while its == 0 or tt < budget_s:
            dn, dt, w = arm.time([seeds_of_t(t0 + its)], [BASE_RNG_SEED_BENCH + t0 + its], w, lr)
            n, tt, its = n + dn, tt + dt, its + 1
    finally:
        arm.close()
    one = OracleArm(gd, cfg, kind, 1)
    try:
        sl = seeds_of_t(t0)[: max(1, len(seeds_of_t(t0)) // P)]
        one.time([sl], [BASE_RNG_SEED_BENCH - 1], weights, lr)
        n1, t1, _ = one.time([sl], [BASE_RNG_SEED_BENCH + t0], weights, lr)
    finally:
        one.close()
    gb = len(seeds_of_t(t0))
    return {"value": n / tt, "unit": UNIT, "cores": P, "kind": "oracle",
            "sample": f"{its} oracle iteration(s) of the {gb}-seed global batch (sample+gather+fwd+loss+bwd+SGD, "
                      f"float64 NumPy/SciPy) on the {cfg['name']}-shaped graph: {P} worker processes x 1 BLAS thread, "
                      f"each a contiguous slice of the batch (as ranks), features shared through /dev/shm; {tt:.1f} s",
            "procs": P, "blas_threads_per_proc": 1, "cpu_model": cpu_model(),
            "one_core": {"value": n1 / t1, "unit": UNIT,
                         "sample": f"1 worker process, 1 BLAS thread, one {len(sl)}-seed slice; {t1:.1f} s"}}


BASE_RNG_SEED_BENCH = 0x5EED


def run_reference(args):
    """--impl reference: the CPU oracle on this workload (rank 0 only), with
    the same config and global batch per step as our arm."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_2404_09544_b200.partition import global_batch, rank_slice
    from synth import CONFIGS, epoch_seeds, init_weights
    from synth.store import shared_graph

    cfg = bench_cfg(args)
    gd = shared_graph(cfg, local)
    dims = [gd.d] + [cfg["hidden"]] * (len(cfg["fanouts"]) - 1) + [gd.C]
    w = init_weights(dims, kind=args.kind)
    perm = epoch_seeds(gd.n, 0)
    B = cfg["batch"]

    def seeds_of_t(t):
        lo, _ = rank_slice(t, 0, world, B, gd.n)
        return perm[lo:lo + global_batch(t, world, B, gd.n)]

    P = cpu_cores()
    arm = OracleArm(gd, cfg, args.kind, P)
    try:
        _, _, w = arm.time([seeds_of_t(t) for t in range(args.warmup)],
                           [BASE_RNG_SEED_BENCH + t for t in range(args.warmup)], w, 0.01)
        ts = range(args.warmup, args.warmup + args.steps)
        n, tt, _ = arm.time([seeds_of_t(t) for t in ts], [BASE_RNG_SEED_BENCH + t for t in ts], w, 0.01)
    finally:
        arm.close()
    value = n / tt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tt / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(cfg, gd, world, args.kind),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": P, "kind": "oracle", "procs": P,
                         "blas_threads_per_proc": 1, "cpu_model": cpu_model(),
                         "sample": f"{args.steps} oracle iterations (after {args.warmup} warm-up) of the "
                                   f"{world * B}-seed global batch, {P} worker processes x 1 BLAS thread over "
                                   f"/dev/shm features, float64"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_cfg(args) -> dict:
    from synth import CONFIGS

    cfg = dict(CONFIGS[args.config])
    if args.ratio is not None:
        cfg["ratio"] = args.ratio
    return cfg


def config_of(cfg, gd, world, kind) -> dict:
    """The workload (identical in both arms)."""
    L = len(cfg["fanouts"])
    return {"workload": cfg["name"], "n_nodes": gd.n, "nnz": gd.nnz, "d": gd.d, "classes": gd.C,
            "fanouts": cfg["fanouts"], "batch_per_rank": cfg["batch"], "global_batch": world * cfg["batch"],
            "cache_ratio": cfg["ratio"], "kind": kind, "hidden": cfg["hidden"], "layers": L,
            "parallelism": f"dp{world}",
            "l2": ("inputs > L2, no flush (feature table %.0f MB, CSR %.0f MB)" if gd.n * gd.stride * 4 > 126e6 else
                   "feature table %.0f MB, CSR %.0f MB: may be L2-resident between steps (no flush)") % (
                gd.n * gd.stride * 4 / 1e6, gd.nnz * 4 / 1e6)}


def algorithmic(seg: str, sizes, cfg, dims, stride, prec, peaks):
    """(bound, amount per launch, unit, peak) for a timeline segment.

    sizes: dict of per-step averages (n[h], nnz[h], U[h] distinct referenced
    src rows per block, hits/misses).  Formulas: DESIGN.md §5 / SURVEY §8(d)."""
    L = len(cfg["fanouts"])
    n, nnz, U = sizes["n"], sizes["nnz"], sizes["U"]
    name, _, lay = seg.partition(".l")
    if name.startswith("pf_"):  # the prefetch stream's sample / gather
        name = name[3:]
    if name == "gather":
        rowb = stride * 4
        lvl = int(sizes.get("x_level", L))
        ld16x = (dims[0] + 1 + 7) & ~7
        if lvl < 0 and sizes.get("fwd16"):  # whole table cached, layer 1 on bf16 copies: F_L rows resolved only
            by = n[L] * 12  # (the layer-1 aggregation copies the dst prefix's bf16 rows, spmm_fwd.l1)
        elif lvl < 0:  # whole table cached, layer-1 GEMMs gather H_dst from it: F_L rows resolved, none copied
            by = n[L] * 12
        elif lvl < L:  # whole table cached: rows of F_{L-1} copied, every F_L row resolved to its cache row
            by = 2 * n[lvl] * rowb + n[L] * 12
            if sizes.get("dw16"):  # + their bf16 copy with the ones column (layer-1 bf16 dW)
                by += n[lvl] * ld16x * 2
        else:
            by = sizes["hits"] * rowb + n[L] * rowb + n[L] * 8
        host = sizes["misses"] * rowb  # zero-copy reads of pinned host rows (Eq.6's transfer)
        if host and peaks.get("host") and host / peaks["host"] > by / peaks["hbm"]:
            return "host-link", host, "GB/s", peaks["host"]
        return "hbm", by, "GB/s", peaks["hbm"]
    if name == "sample":
        by = sum(n[h] * 16 + nnz[h] * 12 for h in range(L))
        return "hbm", by, "GB/s", peaks["hbm"]
    i = int(lay) if lay else 0
    h = L - i
    d_in, d_out = dims[i - 1], dims[i]
    K = 2 * d_in
    # bytes per element of what the step actually stores (reading Q30/Q31):
    # the layer-1 aggregation reads the bf16 table, the hidden H^j / dL/dH^j
    # (j <= L-2) are bf16
    b16 = sizes.get("bf16act", False)
    src_b = 2 if (i == 1 and sizes.get("table16", False)) or (b16 and 2 <= i <= L - 1) else 4
    dw16 = i == 1 and sizes.get("dw16", False)  # layer 1's dW over bf16 operands (reading Q32)
    fwd16 = i == 1 and sizes.get("fwd16", False)  # and its forward GEMM (reading Q33): A^1 kept as bf16 only
    hid16 = 2 <= i <= L - 1 and sizes.get("hid16", False)  # hidden layers' forward GEMM on bf16 (reading Q34)
    if name == "spmm_fwd":
        by = U[h] * d_in * src_b + (0 if fwd16 else n[h] * ((d_in + 3) & ~3) * 4) + nnz[h] * 4 + (n[h] + 1) * 4
        if dw16:  # + the bf16 copy of A^1
            by += n[h] * ((d_in + 7) & ~7) * 2
        if fwd16:  # + the dst rows' own bf16 table rows copied into X16 (with the ones column)
            by += n[h] * ((d_in + 7) & ~7) * 2 + n[h] * ((d_in + 1 + 7) & ~7) * 2
        if hid16:  # + the bf16 copy of A^i
            by += n[h] * ((d_in + 31) & ~31) * 2
        return "hbm", by, "GB/s", peaks["hbm"]
    if name == "spmm_bwd":
        # dA read, block CSR + owner masks read, every dH_src row written once,
        # and the n_dst rows the dX GEMM wrote read back for accumulation
        ld = (d_in + 3) & ~3
        gb = 2 if (b16 and i - 1 <= L - 2) else 4
        by = n[h] * d_in * 4 + nnz[h] * 4 + (n[h] + 1) * 8 + n[h + 1] * ld * gb + n[h] * ld * gb
        return "hbm", by, "GB/s", peaks["hbm"]
    if name in ("tail_a", "tail_b"):
        # fused output layer (tail.cu).  a: self + sampled neighbour rows of
        # H^{L-1} read, aggregates, logits and dlogits written, the dH rows
        # of the seeds and of every owner edge written, dA saved.  b: dA and
        # the non-owner edges' dH rows read-modify-written, [H | A] and dz
        # read for dW.
        ld = (d_in + 3) & ~3
        if name == "tail_a":
            by = (U[h] + n[h]) * d_in * 4 + n[h] * ld * 4 + 2 * n[h] * ((d_out + 3) & ~3) * 4 \
                + n[h + 1] * ld * 4 + n[h] * d_in * 4 + nnz[h] * 4
        else:
            rep = max(0, nnz[h] - (n[h + 1] - n[h]))
            by = n[h] * d_in * 4 + rep * ld * 8 + n[h] * (2 * d_in + d_out) * 4
        return "hbm", by, "GB/s", peaks["hbm"]
    if name == "relu_mask":
        return "hbm", 3 * n[h] * ((d_out + 3) & ~3) * 4, "GB/s", peaks["hbm"]
    ld_in, ld_out = (d_in + 3) & ~3, (d_out + 3) & ~3
    out16 = b16 and i <= L - 2  # H^i (and dL/dH^i) kept as bf16, fp32 rows only for the next dst prefix
    if name == "gemm_fwd":
        fl = 2.0 * n[h] * K * d_out
        by = n[h] * (K * 4 if not (fwd16 or hid16) else (K + 1) * 2 if fwd16 else K * 2) + (n[h] * ld_out * 2 + n[h - 1] * ld_out * 4 if out16 else n[h] * ld_out * 4)
    elif name == "gemm_dx":
        fl = 2.0 * n[h] * K * d_out
        by = n[h] * d_out * (2 if hid16 and sizes.get("hid16_dw") else 4) + n[h] * ld_in * (
            2 if b16 and i - 1 <= L - 2 else 4) + n[h] * ld_in * 4
    elif name == "gemm_dw":
        fl = 2.0 * n[h] * (K + 1) * d_out
        by = n[h] * (K * 4 if not dw16 else (K + 1) * 2) + n[h] * d_out * (2 if out16 else 4)
        if hid16 and sizes.get("hid16_dw"):  # dW over [H16 | A16] and G16
            # G16 from the fused output layer (tail16), or converted from the fp32 G here (+ db)
            by = n[h] * K * 2 + n[h] * d_out * (2 if (sizes.get("tail16") and i == L - 1) else 4 + 2 + 2)
    else:
        return None
    if prec == "fp32":
        return "alu", fl, "TFLOP/s", FP32_SIMT_TFLOPS
    # tensor-core modes: the binding roof is the larger of the two times
    bf16_op = ((dw16 or (hid16 and sizes.get("hid16_dw"))) and name in ("gemm_dw", "gemm_dx")) or (
        (fwd16 or hid16) and name == "gemm_fwd")
    tpeak = peaks["bf16_sust"] * (0.5 if prec == "tf32" and not bf16_op else 1.0)  # tf32 = 1/2 bf16 rate (guide)
    if by / (peaks["hbm"] * 1e9) >= fl / (tpeak * 1e12):
        return "hbm", by, "GB/s", peaks["hbm"]
    return "tensor", fl, "TFLOP/s", tpeak


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2404_09544_b200 import gnnv
    from synth import BASE_RNG_SEED, epoch_seeds, init_weights
    from synth.store import host_bytes, shared_graph

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = bench_cfg(args)
    # one host copy of the graph per box (/dev/shm): local rank 0 generates
    # it (or finds it), every rank maps it; the feature table is then
    # page-locked in place by gnnv_graph_load
    t_gen = time.perf_counter()
    gd = shared_graph(cfg, local)
    t_gen = time.perf_counter() - t_gen
    gnnv.load()
    comm = None
    if world > 1:
        obj = [gnnv.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = gnnv.Comm(rank, world, obj[0], local)
    torch.cuda.synchronize()
    mem = {}
    free0, total_mem = torch.cuda.mem_get_info()
    g = gnnv.Graph.from_data(gd, device=local)
    mem["csr_labels"] = free0 - torch.cuda.mem_get_info()[0]
    placement = gnnv.PLACE_SHARDED if args.placement == "sharded" else gnnv.PLACE_REPLICA
    policy = {"none": gnnv.POLICY_NONE, "degree": gnnv.POLICY_DEGREE, "fifo": gnnv.POLICY_FIFO,
              "lru": gnnv.POLICY_LRU}[args.policy]
    free1 = torch.cuda.mem_get_info()[0]
    cache = gnnv.Cache(g, cfg["ratio"], policy=policy, placement=placement, comm=comm)
    mem["cache_build"] = free1 - torch.cuda.mem_get_info()[0]
    dims = [gd.d] + [cfg["hidden"]] * (len(cfg["fanouts"]) - 1) + [gd.C]
    kind = gnnv.KIND_SAGE if args.kind == "sage" else gnnv.KIND_GCN
    prec = {"fp32": gnnv.PREC_FP32, "bf16": gnnv.PREC_BF16, "tf32": gnnv.PREC_TF32}[args.prec]
    w = init_weights(dims, kind=args.kind)
    B = cfg["batch"]
    free2 = torch.cuda.mem_get_info()[0]
    tr = gnnv.Trainer(g, cache, dims, cfg["fanouts"], B, w, kind=kind, prec=prec, comm=comm)
    tr.set_locality(args.locality_bias)
    bf16act = tr.bf16act()  # TF32 SAGE, L >= 3: the hidden H^i / dL/dH^i kept as bf16 (reading Q30)
    bf16tab = tr.table16()  # whole-table TF32 SAGE: layer 1 aggregates a bf16 copy of the table (reading Q31)
    # the step runs on a high-priority stream; the trainer's prefetch stream
    # has the lowest priority (Eq.4 overlap without delaying the step)
    stream = torch.cuda.Stream(priority=int(os.environ.get("GNNV_STEP_PRIO", "-1")))
    torch.cuda.set_stream(stream)
    lr = 0.01
    # seeds of global iteration t: perm[t*G*B:(t+1)*G*B], rank r takes the r-th B-slice
    from paper_2404_09544_b200.partition import global_batch, iters_per_epoch as _ipe, rank_slice

    perm = epoch_seeds(gd.n, 0)
    iters_per_epoch = _ipe(gd.n, world, B)
    d_perm = torch.as_tensor(perm).cuda()

    def seeds_of(t):
        lo, hi = rank_slice(t, rank, world, B, gd.n)
        if hi <= lo:  # an empty trailing slice of a partial last iteration
            lo, hi = 0, B
        return lo, hi

    pipeline = not args.no_pipeline
    pending = {"t": None}
    # device seeds live in d_perm (ready before the loop): the prefetch is
    # ordered after this idle stream, not after the step in flight
    pf_stream = torch.cuda.Stream()

    def batch(t, host):
        lo, hi = seeds_of(t)
        return (perm[lo:hi] if host else d_perm[lo:hi].data_ptr()), hi - lo

    def run(t, host=False, want_loss=False, prefetch_next=True):
        """One step; with the Eq.4 pipeline the next batch's sample + gather
        is enqueued on the side stream right after this step's compute."""
        seeds, n = batch(t, host)
        if pipeline and pending["t"] != t:
            tr.prefetch(seeds, n, BASE_RNG_SEED + t, on_host=host, stream=pf_stream)
        tr.step(seeds, n, max(n, global_batch(t, world, B, gd.n)), BASE_RNG_SEED + t, lr, on_host=host,
                want_loss=False, stream=stream)
        pending["t"] = None
        if pipeline and prefetch_next:
            s2, n2 = batch(t + 1, host)
            tr.prefetch(s2, n2, BASE_RNG_SEED + t + 1, on_host=host, stream=pf_stream)
            pending["t"] = t + 1
        # the step's loss is read back asynchronously: a ticket now, the value
        # once its copy has landed (one step later), no stream synchronisation
        return tr.loss_async(stream=stream) if want_loss else None

    def drain():
        if pending["t"] is not None:  # consume the trailing prefetch (untimed)
            run(pending["t"], prefetch_next=False)
            torch.cuda.synchronize()

    def step_device(t):
        run(t)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for t in range(args.warmup):
        step_device(t)
    barrier()
    # Gamma (Eq.9-10): device memory of this rank after warm-up
    # (every buffer -- both Eq.4 buffer sets included -- is allocated by now;
    # a step allocates nothing)
    mem["trainer_runtime"] = free2 - torch.cuda.mem_get_info()[0]
    mem["device_used_total"] = total_mem - torch.cuda.mem_get_info()[0]
    # ---------------------------------------------------------- timed region
    # K steps without instrumentation (value); the per-kernel rooflines come
    # from the next K steps, timed the same way with the library's
    # per-segment CUDA events on (those events cost ~4% of a step: they end
    # the programmatic-dependent-launch overlap at every segment boundary)
    t0_steps = args.warmup
    tr.timeline(False)
    clocks = ClockSampler(local)
    clocks.start()
    dyn0 = cache.counters() if args.policy in ("fifo", "lru") else None
    launches0 = gnnv.launch_count()
    barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for i, t in enumerate(range(t0_steps, t0_steps + args.steps)):
        step_device(t)
        if i + 1 < args.steps:
            evs[i + 1].record(stream)
    # the batch prefetched during the last timed step belongs to the region:
    # close it only when that prefetch is done too
    tr.join_prefetch(stream)
    evs[-1].record(stream)
    barrier()
    launches = gnnv.launch_count() - launches0
    # dynamic cache: hit rate of the batches gathered during the timed region
    # (prefetches included), from the cache's own cumulative counters
    dyn = None
    if dyn0 is not None:
        d1 = cache.counters() - dyn0
        dyn = {"hits": int(d1[0]), "misses": int(d1[1]), "replaced": int(d1[2]),
               "hit_rate": float(d1[0]) / max(1, int(d1[0] + d1[1]))}
    clk = clocks.stop()
    ms_total = max_over_ranks(evs[0].elapsed_time(evs[-1]))
    ms_per_step = ms_total / args.steps
    step_ms = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)])
    step_stats = {"median_ms": float(np.median(step_ms)), "p90_ms": float(np.percentile(step_ms, 90)),
                  "min_ms": float(step_ms.min()), "max_ms": float(step_ms.max()),
                  "note": "per-step CUDA events on the step stream (rank 0); the last step also waits for the "
                          "batch it prefetched"}
    value = world * B * args.steps / (ms_total / 1000.0)
    # ------------------------------------- instrumented pass (rooflines)
    tr.timeline(True)
    barrier()
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    for t in range(t0_steps + args.steps, t0_steps + 2 * args.steps):
        step_device(t)
    tr.join_prefetch(stream)
    ev3.record(stream)
    barrier()
    ms_instr = max_over_ranks(ev2.elapsed_time(ev3)) / args.steps
    segs = tr.timeline_read()
    tr.timeline(False)
    # ------------------------------------------------------- e2e (host I/O)
    # host seeds copied in (inside the prefetch / step call) and the loss read
    # back every step through the public API
    drain()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_e2e0 = time.perf_counter()
    e0.record(stream)
    loss = None
    prev = None
    for t in range(t0_steps, t0_steps + args.steps):
        ticket = run(t, host=True, want_loss=True)
        if prev is not None:
            loss = tr.loss_result(prev)  # step t-1's loss on the host (device -> host read every step)
        prev = ticket
    loss = tr.loss_result(prev)
    tr.join_prefetch(stream)
    e1.record(stream)
    barrier()
    wall_e2e = time.perf_counter() - t_e2e0
    ms_e2e = max_over_ranks(e0.elapsed_time(e1))
    value_e2e = world * B * args.steps / (ms_e2e / 1000.0)
    drain()
    # ------------------------------------------- sizes of the timed steps
    nsz = min(args.steps, 8)
    blk = gnnv.Blocks(g, B, cfg["fanouts"])
    blk.set_locality(cache, args.locality_bias)
    L = len(cfg["fanouts"])
    acc = {"n": np.zeros(L + 1), "nnz": np.zeros(L), "U": np.zeros(L), "hits": 0.0, "misses": 0.0}
    cv = cache.info()
    slot_map = torch.empty(gd.n, dtype=torch.int32, device="cuda")
    d2d(slot_map, cv.d_slot, 4 * gd.n)
    for t in range(t0_steps, t0_steps + nsz):
        lo, hi = seeds_of(t)
        blk.sample(d_perm[lo:hi].data_ptr(), hi - lo, BASE_RNG_SEED + t, stream=stream)
        views = blk.info(sync=True, stream=stream)
        for h, v in enumerate(views):
            acc["n"][h] += v.n_dst
            acc["nnz"][h] += v.nnz
            if v.nnz:
                idx = torch.empty(int(v.nnz), dtype=torch.int32, device="cuda")
                d2d(idx, v.d_indices, 4 * int(v.nnz))
                acc["U"][h] += int(torch.unique(idx).numel())
        nL = int(views[-1].n_src)
        acc["n"][L] += nL
        FL = torch.empty(nL, dtype=torch.int32, device="cuda")
        d2d(FL, views[-1].d_src_global, 4 * nL)
        hit = int((slot_map[FL.long()] >= 0).sum().item())
        acc["hits"] += hit
        acc["misses"] += nL - hit
    sizes = {k: (v / nsz) for k, v in acc.items()}
    sizes["x_level"] = tr.x_level()
    sizes["bf16act"] = tr.bf16act()
    sizes["table16"] = tr.table16()
    sizes["dw16"] = tr.dw16()
    sizes["fwd16"] = tr.fwd16()
    sizes["hid16"] = L >= 3 and bool(tr.aggregate16(2)[0])
    sizes["hid16_dw"] = L >= 3 and bool(tr.gradient16(L - 1)[0])
    sizes["tail16"] = tr.tail16()
    peaks = load_peaks()
    if sizes["misses"] > 0:
        peaks["host"] = measure_host_link()
    # the committed captures are of the default knobs (degree cache, no
    # locality bias, replicated, SAGE) at a given config, ratio and precision
    default_cfg = (args.locality_bias == 0 and args.placement == "replica" and args.kind == "sage"
                   and args.policy == "degree")
    traffic = load_traffic(f"{cfg['name']}@{float(cfg['ratio'])}/{args.prec}") if default_cfg else {}
    # dominant kernel segment of the timed region
    seg_ms = {k: v[0] / max(1, v[1]) for k, v in segs.items()}
    seg_tot = {k: v[0] for k, v in segs.items()}
    ranked = sorted(seg_tot.items(), key=lambda kv: -kv[1])
    # main-stream segments tile the step; pf_* run on the side stream,
    # overlapped with them (Eq.4), so they are not on the critical path
    main_tot = sum(v for k, v in seg_tot.items() if not k.startswith("pf_"))
    roofline = None
    rooflines = {}
    for name, tot in ranked:
        a = algorithmic(name, sizes, cfg, dims, gd.stride, args.prec, peaks)
        if a is None:
            continue
        bound, amount, unit, peak = a
        avg_ms = seg_ms[name]
        achieved = amount / (avg_ms / 1000.0) / (1e9 if unit == "GB/s" else 1e12)
        r = {"kernel": name, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
             "frac": achieved / peak, "traffic": traffic.get(name[3:] if name.startswith("pf_") else name),
             "avg_ms": avg_ms,
             "share_of_step": tot / max(1e-9, main_tot),
             "algorithmic_per_launch": amount}
        if name.startswith("pf_"):
            r["overlapped"] = True
        if name.startswith("spmm_fwd."):
            # the edge-visit view -- every sampled edge reads a
            # whole source row (re-reads of rows shared by several dst rows
            # included) plus the output rows -- next to the distinct-row one
            i = int(name.split(".l")[1])
            h = len(cfg["fanouts"]) - i
            d_in = dims[i - 1]
            eb = 2 if (i == 1 and sizes["table16"]) or (sizes["bf16act"] and 2 <= i <= L - 1) else 4
            ob = ((d_in + 3) & ~3) * 4 * (0 if (i == 1 and sizes["fwd16"]) else 1) + (
                ((d_in + 7) & ~7) * 2 if (i == 1 and sizes["dw16"]) else 0)  # fp32 and / or bf16 A rows
            ev = sizes["nnz"][h] * d_in * eb + sizes["n"][h] * ob
            r["edge_visit_bytes"] = ev
            r["edge_visit_frac"] = ev / (avg_ms / 1000.0) / 1e9 / peaks["hbm"]
        rooflines[name] = r
    # the dominant kernel of the critical path: the largest step-stream
    # segment -- unless the step stream spends a quarter of its time waiting
    # for the Eq.4 prefetch (host-miss-bound configs: the zero-copy gather
    # over PCIe is then the critical path), in which case the prefetch's
    # larger segment
    wait = seg_tot.get("wait_prefetch", 0.0)
    pf_bound = wait > 0.25 * main_tot or (
        "pf_gather" in rooflines and rooflines["pf_gather"]["bound"] == "host-link"
        and rooflines["pf_gather"]["avg_ms"] > 0.5 * (main_tot / max(1, args.steps)))
    for name, tot in ranked:
        if name not in rooflines:
            continue
        if name.startswith("pf_") != pf_bound:
            continue
        if pf_bound and name == "pf_sample" and "pf_gather" in rooflines and \
                seg_tot["pf_gather"] >= 0.5 * seg_tot["pf_sample"]:
            continue  # the sampler's overlapped time is stretched by its low priority
        roofline = dict(rooflines[name], critical_path="prefetch" if pf_bound else "step")
        break
    # north_star's "per-iteration gather+SpMM" against HBM: algorithmic bytes
    # of the gather and every aggregation segment over their summed times
    gs = [k for k in rooflines if k.split(".")[0] in ("gather", "pf_gather", "spmm_fwd", "spmm_bwd")]
    gather_spmm = None
    if gs:
        by = sum(rooflines[k]["algorithmic_per_launch"] for k in gs)
        ms = sum(rooflines[k]["avg_ms"] for k in gs)
        gather_spmm = {"segments": gs, "bytes": by, "ms": ms, "achieved": by / ms / 1e6, "peak": peaks["hbm"],
                       "unit": "GB/s", "frac": by / ms / 1e6 / peaks["hbm"],
                       "note": "pf_gather, when present, is timed while overlapped with the step"}
    # -------------------------------------------------------- CPU baseline
    # after every GPU measurement (rank 0; the other ranks wait at the barrier)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        from paper_2404_09544_b200.partition import global_batch as _gb

        def seeds_of_t(t):
            lo, _ = rank_slice(t, 0, world, B, gd.n)
            return perm[lo:lo + max(1, _gb(t, world, B, gd.n))]

        cpu = oracle_baseline(gd, cfg, args.kind, perm, seeds_of_t, t0_steps, w, lr,
                              budget_s=float(os.environ.get("GNNV_CPU_BUDGET_S", "20")))
    if world > 1:
        dist.barrier()
    # Gamma of this rank (Eq.9-10): the cache table, the CSR, the runtime
    # buffers; and the estimator's prediction of the same (NEXT-4)
    from paper_2404_09544_b200.estimator import Candidate, Estimator

    cv = cache.info()
    cand = Candidate(n_nodes=gd.n, nnz=gd.nnz, n_attr=gd.d, stride=gd.stride, n_classes=gd.C, batch=B,
                     fanouts=list(cfg["fanouts"]), hidden=cfg["hidden"], ratio=cfg["ratio"],
                     locality_bias=args.locality_bias, policy=args.policy, kind=args.kind)
    try:
        pred = Estimator(coef={}).memory(cand)
    except Exception:
        pred = None
    gamma = {"gamma_cache_gb": cv.bytes / 1e9, "csr_labels_gb": mem["csr_labels"] / 1e9,
             "cache_build_gb": mem["cache_build"] / 1e9, "trainer_runtime_gb": mem["trainer_runtime"] / 1e9,
             "device_used_gb": mem["device_used_total"] / 1e9, "device_total_gb": total_mem / 1e9,
             "host_store_gb": host_bytes(cfg) / 1e9,
             "eq9_10_predicted_gb": ({k: v / 1e9 for k, v in pred.items()} if pred else None),
             "note": "cudaMemGetInfo deltas on this rank (cache_build includes the table; device_used includes the "
                     "CUDA context and torch's allocations)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": {"fp32": "f32", "bf16": "f32+bf16gemm", "tf32": "f32+tf32gemm"}[args.prec] + (
                "+bf16act" if bf16act else "") + ("+bf16table" if bf16tab else "") + (
                "+bf16dw1" if tr.dw16() else "") + ("+bf16fwd1" if tr.fwd16() else "") + (
                "+bf16fwd2" if sizes["hid16"] else ""), "data": "synthetic",
            "config": config_of(cfg, gd, world, args.kind),
            "settings": {"placement": args.placement, "locality_bias": args.locality_bias,
                         "cache_policy": args.policy, "gemm_precision": args.prec,
                         "bf16_intermediates": bf16act, "bf16_table_layer1": tr.table16(),
                         "bf16_dw_layer1": tr.dw16(), "bf16_fwd_layer1": tr.fwd16(),
                         "bf16_fwd_hidden": sizes["hid16"],
                         "gathered_x_mb_per_step": sizes["n"][L] * gd.stride * 4 / 1e6,
                         "pipeline": "eq4-overlap (next batch sample+gather on a side stream)" if pipeline else "off"},
            "step_stats": step_stats,
            "gamma": gamma,
            "epoch_s": iters_per_epoch * ms_per_step / 1000.0,
            "iters_per_epoch": iters_per_epoch,
            "clocks": clk,
            "gpu_launches": int(launches),
            "roofline": roofline,
            "rooflines": rooflines,
            "rooflines_pass": {"steps": args.steps, "ms_per_step": ms_instr,
                               "note": "per-segment CUDA events on the step stream; a second pass of K steps "
                                       "right after the timed one"},
            "gather_spmm": gather_spmm,
            "phases_ms_per_step": {k: v[0] / args.steps for k, v in sorted(segs.items(), key=lambda kv: -kv[1][0])},
            "sizes_per_step": {"frontier": [round(x) for x in sizes["n"]], "edges": [round(x) for x in sizes["nnz"]],
                               "distinct_src": [round(x) for x in sizes["U"]], "cache_hits": sizes["hits"],
                               "cache_misses": sizes["misses"],
                               "x_rows_level": sizes["x_level"]},
            "e2e": {"value": value_e2e, "unit": UNIT, "h2d_bytes_per_step": B * 4, "d2h_bytes_per_step": 8,
                    "ms_per_step": ms_e2e / args.steps, "wall_s": wall_e2e, "last_loss": loss},
            "dynamic_cache": dyn,
            "cpu_baseline": cpu,
            "vs_cpu_baseline": (value / cpu["value"]) if cpu else None,
            "peaks": peaks["src"] + (f"; host link {peaks['host']:.1f} GB/s measured (best of the pinned H2D copy and SM zero-copy reads)"
                                     if peaks.get("host") else ""),
            "graph_gen_s": t_gen,
        }
        print(json.dumps(line), flush=True)
    tr.free()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
