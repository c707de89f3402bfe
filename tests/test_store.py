"""CPU: the shared host store (synth/store.py) -- one copy of a generated
graph per box, mapped read-only by every rank and CPU-baseline worker."""
import os

import numpy as np

from synth import CONFIGS, make_graph
from synth.store import host_bytes, open_store, shared_graph, store_key, store_path


def test_store_round_trip(tmp_path):
    cfg = CONFIGS["mini"]
    ref = make_graph(cfg)
    gd = shared_graph(cfg, root=str(tmp_path))
    assert os.path.isdir(store_path(cfg, str(tmp_path)))
    for a, b in ((gd.indptr, ref.indptr), (gd.indices, ref.indices), (gd.feats, ref.feats),
                 (gd.labels, ref.labels)):
        assert isinstance(a, np.memmap)
        assert a.dtype == b.dtype and a.shape == b.shape
        np.testing.assert_array_equal(a, b)
    assert (gd.n, gd.d, gd.C, gd.name) == (ref.n, ref.d, ref.C, ref.name)
    assert gd.feats.ctypes.data % 16 == 0  # gnnv_graph_load registers it in place
    assert not gd.indices.flags.writeable
    # a second process (rank) maps the same store without regenerating it
    again = open_store(store_path(cfg, str(tmp_path)))
    np.testing.assert_array_equal(again.indices, ref.indices)
    assert sum(f.stat().st_size for f in os.scandir(store_path(cfg, str(tmp_path)))) >= host_bytes(cfg)


def test_store_key_tracks_generator_fields():
    a = dict(CONFIGS["mini"])
    b = dict(a, beta=0.6)
    c = dict(a, hidden=999)  # not a generator field
    assert store_key(a) != store_key(b)
    assert store_key(a) == store_key(c)


def test_store_falls_back_without_root(tmp_path):
    gd = shared_graph("mini", root=str(tmp_path / "missing"))
    assert not isinstance(gd.indices, np.memmap)
    assert gd.n == CONFIGS["mini"]["n"]
