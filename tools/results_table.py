"""Markdown rows for DESIGN.md §6 / README.md from the committed per-config
bench lines (profiles/r02_bench_<config>@<ratio>.json) and ncu summaries
(profiles/r02_ncu_traffic_<config>@<ratio>.json).

    python tools/results_table.py
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFGS = [("cora", "0.2", 0), ("arxiv", "0.5", 1), ("reddit", "0.1", 2), ("reddit", "1.0", 2), ("products", "1.0", 3),
        ("papers100m", "1.0", 4)]


def main():
    print("| config | seeds/s | ms/step (median, p90) | epoch s | e2e seeds/s | critical path: kernel, bound, frac | "
          "gather+SpMM frac | DRAM per serial step (ncu) | Γ_cache / device used | oracle (P procs) |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for name, ratio, idx in CFGS:
        tag = f"{name}@{ratio}"
        p = os.path.join(ROOT, "profiles", f"r02_bench_{tag}.json")
        if not os.path.exists(p):
            continue
        d = json.load(open(p))
        r = d["roofline"]
        st = d.get("step_stats") or {}
        g = d.get("gamma") or {}
        cb = d.get("cpu_baseline") or {}
        nt = os.path.join(ROOT, "profiles", f"r02_ncu_traffic_{tag}.json")
        dram = "—"
        if os.path.exists(nt):
            segs = json.load(open(nt))["segments"]
            dram = f"{sum(v['dram_bytes'] for v in segs.values()) / 1e9:.2f} GB"
        print(f"| {tag} (configs[{idx}]) | {d['value'] / 1e6:.2f} M | {d['ms_per_step']:.3f} "
              f"({st.get('median_ms', float('nan')):.3f}, {st.get('p90_ms', float('nan')):.3f}) | "
              f"{d.get('epoch_s', float('nan')):.3f} | {d['e2e']['value'] / 1e6:.2f} M | "
              f"{r['kernel']}, {r['bound']}, {r['frac']:.2f} | {d['gather_spmm']['frac']:.2f} | {dram} | "
              f"{g.get('gamma_cache_gb', float('nan')):.2f} / {g.get('device_used_gb', float('nan')):.1f} GB | "
              f"{cb.get('value', float('nan')):.0f} ({cb.get('cores', '?')}) |")


if __name__ == "__main__":
    main()
