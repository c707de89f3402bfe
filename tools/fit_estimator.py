"""Fit the gray-box estimator (NEXT-4) on profile records and report its
leave-one-out accuracy.

    python tools/fit_estimator.py profiles/r01_estimator_records.jsonl > profiles/r01_estimator_fit.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2404_09544_b200.estimator import Candidate, fit, frontier_sizes  # noqa: E402


def deg_hist(name):
    from synth import make_graph

    gd = make_graph(name, with_feats=False)
    d = np.minimum(np.diff(gd.indptr), 64)
    return (np.bincount(d, minlength=65) / gd.n).tolist()


def main():
    recs = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
    hists = {}
    for r in recs:  # the graph statistic the sweep did not record
        if not r["candidate"].get("deg_hist"):
            if r["graph"] not in hists:
                hists[r["graph"]] = deg_hist(r["graph"])
            r["candidate"]["deg_hist"] = hists[r["graph"]]
    full = fit(recs)
    rows = []
    for i, r in enumerate(recs):
        est = fit(recs[:i] + recs[i + 1:])  # leave one out
        c = Candidate(**r["candidate"])
        pred_f = frontier_sizes(c, *est.overlap)
        t = est.phase_times(c, r["hit"])
        rows.append({
            "graph": r["graph"], "batch": c.batch, "fanouts": list(c.fanouts), "ratio": c.ratio,
            "bias": c.locality_bias, "policy": c.policy,
            "V_i": [r["frontier"][-1], pred_f[-1]],
            "serial_ms": [r["serial_ms"], 1e3 * sum(t.values())],
            "pipelined_ms": [r["pipelined_ms"], 1e3 * est.step_time(c, r["hit"], True)],
        })
    err = lambda k: float(np.mean([abs(x[k][1] - x[k][0]) / x[k][0] for x in rows]))
    out = {"fit_all": json.loads(full.to_json()),
           "loo_mape": {"V_i": err("V_i"), "serial_ms": err("serial_ms"), "pipelined_ms": err("pipelined_ms")},
           "loo": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
