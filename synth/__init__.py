"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds ONLY input generators (graphs, features, labels, seed
permutations, initial weights).  It contains none of the method's
arithmetic (no sampling, relabelling, caching, aggregation or training):
both `oracle/` and `paper_2404_09544_b200/` may import it, neither imports
the other.
"""
from .graphs import (  # noqa: F401
    BASE_RNG_SEED,
    CONFIGS,
    GraphData,
    chung_lu_graph,
    csr_from_edges,
    epoch_seeds,
    init_weights,
    make_graph,
    make_features,
    make_labels,
    tiny_graph,
    row_stride,
)
