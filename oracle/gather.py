"""Feature retrieval for the sampled rows (oracle side).

Paper: Algorithm 1 line 3 MemcpyHtoD(G_i); transmission
abstraction P:268-270 ("the device cache figures out which part of the
mini-batch has been cached.  The remaining part is filtered out from the
host and transferred").  Wherever a row comes from (cache, peer, host), the
value is the vertex's feature row h^0_v: X[i,:] = feat[F_L[i], :].
Bit-exact copy; the stored row stride (padding zero) is kept.
"""
from __future__ import annotations

import numpy as np


def gather_rows(feats: np.ndarray, rows: np.ndarray) -> np.ndarray:
    return np.asarray(feats)[np.asarray(rows, dtype=np.int64)].copy()
