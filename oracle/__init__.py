"""CPU oracle for the GNNavigator (arXiv 2404.09544) mini-batch hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import or execute
anything in this package.  The product path (`paper_2404_09544_b200/`) never
imports it and shares no code with it; the only common module is `synth/`
(seeded input generators, none of the method's arithmetic).

Every function is a plain, slow, obviously-correct restatement of the paper's
step (float64 for floating point), citing the passage it follows
(`P:n` = /root/reference/PAPER.md line n, `S:n` = SPEC.md line n).  Readings
where the paper is silent are listed in DESIGN.md §3 as Q1..Q21.

Pins (tests/test_oracle_*.py, `-m "not gpu"`): Random123 known-answer vectors
for Philox; exhaustive enumeration of Floyd's draw tuples; networkx L-hop BFS
for the exhaustive-fanout case; SPEC worked examples; brute-force dense
adjacency for aggregation; torch float64 autograd and central finite
differences for layer/loss/backward.

Parity unpinned: WHICH k-subset a node draws is fixed by this repo's own
definition (Philox key layout + Floyd), not by the paper; only the
distribution (uniform over k-subsets) is pinned.
"""
from .philox import philox4x32_10, draw, uniform_int  # noqa: F401
from .sampler import floyd_positions, sample_hop_positions, sample_blocks, Block  # noqa: F401
from .cache import cache_capacity, degree_rank, cache_slots, access_counts  # noqa: F401
from .gather import gather_rows  # noqa: F401
from .layers import (  # noqa: F401
    agg_matrix, layer_fwd, layer_bwd, ce_loss, sgd_update, train_step, forward_all,
    flop_count,
)
