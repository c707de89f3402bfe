"""Gray-box performance estimator: the paper's Eq.4-10
and Eq.12 with the learned parts fitted on this backend's own
per-phase B200 profiles (tools/profile_sweep.py).

White box (the paper's equations):
  Eq.4   T = n_iter * max(t_sample + t_transfer, t_replace + t_compute)
         (here the left branch is the Eq.4 prefetch stream and
         the right one the step stream, so the max is literal)
  Eq.5   t_replace  = f_replace(r|V|, |V_i|(1-hit))
  Eq.6   t_transfer = f_transfer(n_attr |V_i| (1-hit))   (+ the hits' HBM copy on B200)
  Eq.7   t_sample   = f_sample(|V_i| - |B0|)
  Eq.8   t_compute  = f_compute(|V_i|, M)
  Eq.9-10 Gamma = Gamma_model + Gamma_cache + Gamma_runtime
  Eq.12  E|V_i| = f_overlapping(|B0| prod_l (1 + k^l), p(eta))
Black box (fitted here, reading Q28): every f_* is linear in the physical
quantity the paper names -- bytes for the memory-bound phases, sampled edges
for the sampler, flops and activation bytes for compute -- with
non-negative coefficients (seconds per unit on this GPU); f_overlapping is
the per-hop keep fraction 1 / (1 + a x^b) of the Eq.12 bound, x = n_h k_h / N.
Accuracy (Eq.11) is out of scope (no datasets).
"""
from __future__ import annotations

import dataclasses
import json
import math
from typing import Dict, List, Sequence

import numpy as np


@dataclasses.dataclass
class Candidate:
    """A point of the design space (the knobs of P:220-227 / reading Q21)."""
    n_nodes: int
    nnz: int
    n_attr: int
    stride: int
    n_classes: int
    batch: int
    fanouts: Sequence[int]
    hidden: int
    ratio: float
    locality_bias: float = 0.0
    policy: str = "degree"
    kind: str = "sage"
    # graph statistic: P(deg = d) for d < 64 and P(deg >= 64) (65 bins) --
    # min(k, deg) picks per node (Eq.2) need the low-degree mass
    deg_hist: Sequence[float] = ()

    def dims(self) -> List[int]:
        L = len(self.fanouts)
        return [self.n_attr] + [self.hidden] * (L - 1) + [self.n_classes]

    def n_params(self) -> int:
        d = self.dims()
        mult = 2 if self.kind == "sage" else 1
        return sum(mult * d[i] * d[i + 1] + d[i + 1] for i in range(len(d) - 1))


def eq12_bound(batch: int, fanouts: Sequence[int], n: int) -> List[float]:
    """Frontier sizes without overlap: n_{h+1} = min(N, n_h (1 + k_h)) (Eq.12, tau = 1)."""
    out = [float(batch)]
    for k in fanouts:
        out.append(min(float(n), out[-1] * (1 + k)))
    return out


def picks_per_node(c: Candidate, k: int, hop: int) -> float:
    """E[min(k, deg)] (Eq.2's min(k, |N(v)|)): seeds are uniform vertices,
    later frontier vertices were reached along edges (size-biased degree)."""
    if not c.deg_hist:
        return float(k)
    p = np.asarray(c.deg_hist, float)
    d = np.arange(len(p), dtype=float)
    if hop > 0:
        tail_mean = 2.0 * c.nnz / c.n_nodes  # unused when k < 64: the tail picks k anyway
        w = p * np.where(d < len(p) - 1, d, max(tail_mean, len(p) - 1))
        p = w / w.sum()
    return float((p * np.minimum(d, k)).sum() + 0.0)


def frontier_sizes(c: Candidate, a: float, b: float, g: float = 0.0) -> List[float]:
    """E|F_h| via f_overlapping (Eq.12): hop h draws n_h E[min(k, deg)]
    neighbours, of which a fraction 1/(1 + a x^b m^g) are new, x = n_h k_h / N
    the collision pressure and m = nnz/N the mean degree (graph shape)."""
    out = [float(c.batch)]
    m = c.nnz / float(c.n_nodes)
    for h, k in enumerate(c.fanouts):
        n = out[-1]
        x = n * k / float(c.n_nodes)
        keep = 1.0 / (1.0 + a * x ** b * m ** g)
        out.append(min(float(c.n_nodes), n + n * picks_per_node(c, k, h) * keep))
    return out


def edge_counts(c: Candidate, sizes: Sequence[float]) -> List[float]:
    """Sampled edges per hop: each dst row keeps min(k, deg) ~ k picks."""
    return [sizes[h] * k for h, k in enumerate(c.fanouts)]


def flops(c: Candidate, sizes: Sequence[float], edges: Sequence[float]) -> float:
    """Forward+backward flops of the step (3x the forward GEMMs, SPEC S:341 aggregation terms)."""
    d = c.dims()
    L = len(c.fanouts)
    f = 0.0
    for i in range(1, L + 1):
        h = L - i
        K = (2 if c.kind == "sage" else 1) * d[i - 1]
        f += 3 * 2.0 * sizes[h] * K * d[i] + 2 * edges[h] * d[i - 1]
    return f


def act_bytes(c: Candidate, sizes: Sequence[float]) -> float:
    """Activation bytes written and read per step (fp32), the compute phase's HBM traffic."""
    d = c.dims()
    L = len(c.fanouts)
    return float(sum(4.0 * sizes[L - i] * (2 * d[i - 1] + 2 * d[i]) for i in range(1, L + 1)))


def features(c: Candidate, hit: float, sizes: Sequence[float]) -> Dict[str, float]:
    """The physical quantities Eq.5-8 depend on, for one candidate."""
    L = len(c.fanouts)
    VL = sizes[L]
    edges = edge_counts(c, sizes)
    row = 4.0 * c.stride
    return {
        "sample_edges": float(sum(edges)),                      # Eq.7: |V_i| - |B0| and the edges behind it
        "sample_rows": float(VL - c.batch),
        # NEXT-2's locality-biased sampler sweeps each frontier row's whole
        # adjacency (two ballot passes over the neighbours' cache flags),
        # not only its k picks
        "sample_adj": float(sum(sizes[h] for h in range(L)) * c.nnz / c.n_nodes) if c.locality_bias > 0 else 0.0,
        "transfer_host_bytes": float(VL * (1 - hit) * 4 * c.n_attr),  # Eq.6: n_attr |V_i| (1-hit)
        "transfer_hbm_bytes": float(VL * hit * row),            # the hits' copy out of the device cache
        "replace_rows": float(VL * (1 - hit)) if c.policy in ("fifo", "lru") else 0.0,  # Eq.5
        "compute_flops": flops(c, sizes, edges),                # Eq.8
        "compute_bytes": act_bytes(c, sizes) + 4.0 * sum(edges) * max(c.dims()[:-1]),
    }


PHASES = {
    "sample": ["sample_edges", "sample_rows", "sample_adj"],
    "transfer": ["transfer_host_bytes", "transfer_hbm_bytes"],
    "replace": ["replace_rows"],
    "compute": ["compute_flops", "compute_bytes"],
}


def nnls(A: np.ndarray, y: np.ndarray, iters: int = 2000) -> np.ndarray:
    """Non-negative least squares by projected coordinate descent (small
    problems; the coefficients are seconds per unit, so >= 0)."""
    A = np.asarray(A, float)
    y = np.asarray(y, float)
    x = np.zeros(A.shape[1])
    col = (A * A).sum(axis=0) + 1e-300
    for _ in range(iters):
        for j in range(A.shape[1]):
            r = y - A @ x + A[:, j] * x[j]
            x[j] = max(0.0, float(A[:, j] @ r) / col[j])
    return x


@dataclasses.dataclass
class Estimator:
    coef: Dict[str, np.ndarray]  # per phase: [intercept, coefficients...]
    overlap: tuple = (1.0, 1.0, 0.0)  # f_overlapping (a, b, g)
    # Eq.4 overlap on ONE device: both streams share the SMs and HBM, so a
    # fraction kappa of the shorter branch is not hidden (learned; 0 = Eq.4)
    kappa: float = 0.0

    def phase_times(self, c: Candidate, hit: float) -> Dict[str, float]:
        sizes = frontier_sizes(c, *self.overlap)
        f = features(c, hit, sizes)
        out = {}
        for ph, names in PHASES.items():
            w = self.coef.get(ph)
            if w is None:
                out[ph] = 0.0
                continue
            out[ph] = float(w[0] + sum(w[i + 1] * f[n] for i, n in enumerate(names)))
        if c.policy not in ("fifo", "lru"):
            out["replace"] = 0.0
        return out

    def step_time(self, c: Candidate, hit: float, pipelined: bool = True) -> float:
        t = self.phase_times(c, hit)
        if pipelined:  # Eq.4: the two streams overlap (+ the learned interference)
            a, b = t["sample"] + t["transfer"], t["replace"] + t["compute"]
            return max(a, b) + self.kappa * min(a, b)
        return sum(t.values())

    def epoch_time(self, c: Candidate, hit: float, world: int = 1, pipelined: bool = True) -> float:
        n_iter = math.ceil(c.n_nodes / (world * c.batch))  # reading Q9
        return n_iter * self.step_time(c, hit, pipelined)

    def memory(self, c: Candidate) -> Dict[str, float]:
        """Eq.9-10 on this trainer: params + grads (Gamma_model = 2*4*|Phi|),
        the cache table, and the runtime buffers sized for the Eq.12 bound
        (frontier capacities, two prefetch buffer sets for X and the blocks)."""
        L = len(c.fanouts)
        cap = eq12_bound(c.batch, c.fanouts, c.n_nodes)
        d = c.dims()
        model = 2 * 4.0 * c.n_params()
        cache = math.floor(c.ratio * c.n_nodes) * 4.0 * c.stride
        acts = sum(cap[L - i] * 4.0 * (3 * d[i] + d[i - 1]) for i in range(1, L + 1))
        xbuf = 2 * cap[L] * 4.0 * c.stride
        blocks = 2 * (4.0 * c.n_nodes + sum(cap[h] * (4 * c.fanouts[h] * 3 + 12) for h in range(L)))
        return {"model": model, "cache": cache, "runtime": acts + xbuf + blocks,
                "total": model + cache + acts + xbuf + blocks}

    def to_json(self) -> str:
        return json.dumps({"coef": {k: list(map(float, v)) for k, v in self.coef.items()},
                           "overlap": list(self.overlap), "kappa": self.kappa})


def fit_overlap(records: Sequence[dict]) -> tuple:
    """Fit (a, b, g) of f_overlapping to measured frontier sizes (grid +
    local refinement on the squared log error)."""
    cands = [(Candidate(**r["candidate"]), r["frontier"]) for r in records]

    def loss(a, b, g):
        e = 0.0
        for c, meas in cands:
            pred = frontier_sizes(c, a, b, g)
            for p, m in zip(pred[1:], meas[1:]):
                e += (math.log(p) - math.log(m)) ** 2
        return e

    best = (float("inf"), 1.0, 1.0, 0.0)
    for a in np.geomspace(0.01, 100, 25):
        for b in np.linspace(0.2, 2.0, 10):
            for g in np.linspace(-1.5, 1.5, 7):
                v = loss(a, b, g)
                if v < best[0]:
                    best = (v, float(a), float(b), float(g))
    for it in range(4):
        _, a, b, g = best
        for a2 in np.geomspace(a / 1.5, a * 1.5, 7):
            for b2 in np.linspace(max(0.05, b - 0.2 / (it + 1)), b + 0.2 / (it + 1), 5):
                for g2 in np.linspace(g - 0.25 / (it + 1), g + 0.25 / (it + 1), 5):
                    v = loss(a2, b2, g2)
                    if v < best[0]:
                        best = (v, float(a2), float(b2), float(g2))
    return best[1:]


def fit(records: Sequence[dict]) -> Estimator:
    """Fit every f_* (non-negative linear, with intercept) on profile
    records: {"candidate": {...}, "frontier": [...], "hit": h,
    "phases_ms": {"sample", "transfer", "replace", "compute"}}.  The
    features use the MEASURED frontier sizes (the f_overlapping fit is
    separate), as the black-box parts are learned from profiles."""
    overlap = fit_overlap(records)
    coef = {}
    for ph, names in PHASES.items():
        rows, ys = [], []
        for r in records:
            c = Candidate(**r["candidate"])
            f = features(c, r["hit"], r["frontier"])
            if ph == "replace" and c.policy not in ("fifo", "lru"):
                continue
            rows.append([1.0] + [f[n] for n in names])
            ys.append(r["phases_ms"][ph] * 1e-3)
        if not rows:
            continue
        A = np.asarray(rows)
        scale = np.abs(A).max(axis=0) + 1e-300
        w = nnls(A / scale, np.asarray(ys)) / scale
        coef[ph] = w
    est = Estimator(coef=coef, overlap=overlap)
    # kappa from the measured pipelined steps, given the fitted phases
    num = den = 0.0
    for r in records:
        if "pipelined_ms" not in r:
            continue
        p = r["phases_ms"]
        a, b = (p["sample"] + p["transfer"]) * 1e-3, (p["replace"] + p["compute"]) * 1e-3
        lo = min(a, b)
        num += lo * (r["pipelined_ms"] * 1e-3 - max(a, b))
        den += lo * lo
    est.kappa = max(0.0, num / den) if den > 0 else 0.0
    return est
