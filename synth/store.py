"""One shared host copy of a generated graph per box.

With one process per GPU, every rank needs the same CSR, features and
labels; papers100M-shaped inputs are ~65 GB, so eight private copies (and
eight concurrent generations) do not fit a box.  Instead the first local
process generates the graph once into a directory under /dev/shm (tmpfs,
i.e. RAM), and every process -- GPU ranks and the CPU-baseline workers --
maps the same pages (np.load(..., mmap_mode=...), see open_store).  The feature
table is then page-locked in place by gnnv_graph_load (cudaHostRegister of
the mapping), so misses are zero-copy reads of that one copy.

Layout: <root>/gnnv_<key>/{indptr,indices,feats,labels}.npy + meta.json,
where key hashes the config's generator fields and this package's source
(a store written by another generator version is never reused).  The
directory is written under a temporary name and renamed when complete, so a
reader never sees a half-written store.

This module holds no arithmetic of the method: it only stores and maps the
outputs of synth.graphs.make_graph.
"""
from __future__ import annotations

import hashlib
import json
import os
import shutil
import time
from typing import Callable, Optional

import numpy as np

from .graphs import CONFIGS, GraphData, make_graph

DEFAULT_ROOT = "/dev/shm"
_FIELDS = ("name", "n", "nnz", "d", "C", "beta")


def store_key(cfg: dict) -> str:
    h = hashlib.sha256()
    h.update(json.dumps({k: cfg[k] for k in _FIELDS}, sort_keys=True).encode())
    here = os.path.dirname(os.path.abspath(__file__))
    for f in ("graphs.py", "store.py"):
        h.update(open(os.path.join(here, f), "rb").read())
    return f"{cfg['name']}_{h.hexdigest()[:12]}"


def store_path(cfg: dict, root: str = DEFAULT_ROOT) -> str:
    return os.path.join(root, "gnnv_" + store_key(cfg))


def host_bytes(cfg: dict) -> int:
    """Bytes of one stored copy (CSR + padded features + labels)."""
    stride = (int(cfg["d"]) + 3) & ~3
    n, nnz = int(cfg["n"]), int(cfg["nnz"])
    return (n + 1) * 8 + nnz * 4 + n * stride * 4 + n * 4


def write_store(gd: GraphData, cfg: dict, root: str = DEFAULT_ROOT) -> str:
    final = store_path(cfg, root)
    tmp = f"{final}.tmp{os.getpid()}"
    os.makedirs(tmp, exist_ok=True)
    try:
        for name, arr in (("indptr", gd.indptr), ("indices", gd.indices), ("feats", gd.feats),
                          ("labels", gd.labels)):
            np.save(os.path.join(tmp, name + ".npy"), arr, allow_pickle=False)
        with open(os.path.join(tmp, "meta.json"), "w") as fh:
            json.dump({"n": gd.n, "d": gd.d, "C": gd.C, "name": gd.name}, fh)
        try:
            os.rename(tmp, final)
        except OSError:  # another process completed the same store first
            shutil.rmtree(tmp, ignore_errors=True)
    except BaseException:
        shutil.rmtree(tmp, ignore_errors=True)
        raise
    return final


def open_store(path: str) -> GraphData:
    """Map a complete store (no copy).  The CSR and labels are mapped
    read-only; the feature table is a shared writable mapping (nothing
    writes it) because cudaHostRegister rejects PROT_READ pages (measured on
    the B200 box, tools/probe_hostreg.py: "invalid argument" with or without
    cudaHostRegisterReadOnly, success on a MAP_SHARED read-write mapping)."""
    meta = json.load(open(os.path.join(path, "meta.json")))
    arr = {k: np.load(os.path.join(path, k + ".npy"), mmap_mode="r+" if k == "feats" else "r", allow_pickle=False)
           for k in ("indptr", "indices", "feats", "labels")}
    return GraphData(n=int(meta["n"]), indptr=arr["indptr"], indices=arr["indices"], feats=arr["feats"],
                     d=int(meta["d"]), labels=arr["labels"], C=int(meta["C"]), name=meta["name"])


def shared_graph(cfg, local_rank: int = 0, barrier: Optional[Callable[[], None]] = None,
                 root: str = DEFAULT_ROOT) -> GraphData:
    """The config's graph from the box-wide store: local rank 0 generates it
    if absent (one copy per box), everyone waits on `barrier` (if given) and
    maps it.  Without /dev/shm space the graph is generated privately."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    path = store_path(cfg, root)
    usable = os.path.isdir(root) and os.access(root, os.W_OK)
    if usable and not os.path.isdir(path):
        st = os.statvfs(root)
        usable = st.f_bavail * st.f_frsize > host_bytes(cfg) * 1.05
    if not usable:
        if barrier:
            barrier()
        return make_graph(cfg)
    if local_rank == 0 and not os.path.isdir(path):
        write_store(make_graph(cfg), cfg, root)
    if barrier:
        barrier()
    t0 = time.time()
    while not os.path.isdir(path):  # no barrier: wait for the generating process
        if time.time() - t0 > 3600:
            raise TimeoutError(f"shared graph store {path} not written")
        time.sleep(1.0)
    return open_store(path)


def remove_store(cfg, root: str = DEFAULT_ROOT) -> None:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    shutil.rmtree(store_path(cfg, root), ignore_errors=True)
