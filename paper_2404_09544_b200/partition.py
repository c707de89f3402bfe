"""Seed partitioning across ranks (host logic of the data-parallel path).

Algorithm 1 iterates over i in [0, |V|/|B^0|) mini-batches; with G
ranks the global iteration t covers perm[t*G*B : (t+1)*G*B] of the epoch's
seed permutation and rank r takes the r-th contiguous B-slice (SURVEY
§8(e)); the last iteration of an epoch is partial.
"""
from __future__ import annotations

import math
from typing import Tuple


def iters_per_epoch(n: int, world: int, batch: int) -> int:
    """ceil(N / (G B)) iterations per rank per epoch (reading Q9)."""
    if n < 1 or world < 1 or batch < 1:
        raise ValueError("parameter error")
    return math.ceil(n / (world * batch))


def rank_slice(t: int, rank: int, world: int, batch: int, n: int) -> Tuple[int, int]:
    """[lo, hi) of the epoch permutation that rank `rank` trains on in
    iteration t (t taken modulo the epoch).  May be empty (lo == hi) for the
    trailing ranks of a partial last iteration."""
    if not (0 <= rank < world):
        raise ValueError("parameter error: rank")
    t = t % iters_per_epoch(n, world, batch)
    lo = min(n, t * world * batch + rank * batch)
    hi = min(n, lo + batch)
    return lo, hi


def global_batch(t: int, world: int, batch: int, n: int) -> int:
    """Seeds of global iteration t over all ranks (the loss scale 1/B_global)."""
    t = t % iters_per_epoch(n, world, batch)
    lo = t * world * batch
    return max(0, min(n, lo + world * batch) - lo)
