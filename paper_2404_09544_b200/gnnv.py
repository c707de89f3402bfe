"""Thin ctypes binding of libgnnv (include/gnnv.h).  Argument marshalling only:
every step of the hot path runs in the CUDA kernels of libgnnv.so.  There is
no fallback: if the library is missing, importing the entry points raises.

Names mirror the C API without the `gnnv_` prefix.  Device buffers are given
as torch CUDA tensors (or raw integer pointers); torch is used only for
device memory, streams and process groups.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GNNV_LIB: an alternative build of the same library (A/B timing of two builds)
LIB_PATH = os.environ.get("GNNV_LIB") or os.path.join(_HERE, "libgnnv.so")
MAX_LAYERS = 8

OK, ERR_PARAM, ERR_STATE, ERR_OOM, ERR_CUDA, ERR_COMM, ERR_UNSUPPORTED = range(7)
POLICY_NONE, POLICY_DEGREE, POLICY_FIFO, POLICY_LRU = range(4)
PLACE_REPLICA, PLACE_SHARDED, PLACE_SHARDED_LOCAL = range(3)
KIND_SAGE, KIND_GCN = 0, 1
AGGR_MEAN, AGGR_SUM = 0, 1
ACT_NONE, ACT_RELU = 0, 1
PREC_FP32, PREC_BF16, PREC_TF32 = 0, 1, 2
STATUS_NAMES = {0: "OK", 1: "ERR_PARAM", 2: "ERR_STATE", 3: "ERR_OOM", 4: "ERR_CUDA", 5: "ERR_COMM",
                6: "ERR_UNSUPPORTED"}


class GnnvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class BlockView(C.Structure):
    _fields_ = [("n_dst", C.c_int64), ("n_src", C.c_int64), ("nnz", C.c_int64),
                ("max_dst", C.c_int64), ("max_src", C.c_int64), ("max_nnz", C.c_int64),
                ("d_indptr", C.c_void_p), ("d_indices", C.c_void_p), ("d_src_global", C.c_void_p)]


class GraphView(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("nnz", C.c_int64), ("feat_dim", C.c_int32), ("row_stride", C.c_int32),
                ("n_classes", C.c_int32), ("device", C.c_int32), ("d_indptr", C.c_void_p),
                ("d_indices", C.c_void_p), ("d_labels", C.c_void_p), ("d_host_feats", C.c_void_p)]


class CacheView(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("local_rows", C.c_int64), ("bytes", C.c_int64), ("world", C.c_int32),
                ("rank", C.c_int32), ("placement", C.c_int32), ("d_slot", C.c_void_p), ("d_order", C.c_void_p)]


class LayerDesc(C.Structure):
    _fields_ = [("d_in", C.c_int32), ("d_out", C.c_int32), ("in_stride", C.c_int32), ("kind", C.c_int32),
                ("aggr", C.c_int32), ("act", C.c_int32), ("prec", C.c_int32)]


class ModelDesc(C.Structure):
    _fields_ = [("L", C.c_int32), ("dims", C.c_int32 * (MAX_LAYERS + 1)), ("fanouts", C.c_int32 * MAX_LAYERS),
                ("max_seeds", C.c_int32), ("kind", C.c_int32), ("aggr", C.c_int32), ("prec", C.c_int32)]


class StepTiming(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("sample_ms", "gather_ms", "fwd_ms", "loss_ms", "bwd_ms",
                                          "allreduce_ms", "update_ms", "total_ms")]

    def as_dict(self):
        return {n: float(getattr(self, n)) for n, _ in self._fields_}


class Segment(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("total_ms", C.c_double), ("count", C.c_int32)]


VP, I32, I64, U64, F32, F64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes)
_SIGS = {
    "gnnv_last_error": (C.c_char_p, []),
    "gnnv_version": (C.c_char_p, []),
    "gnnv_set_option": (I32, [C.c_char_p, I32]),
    "gnnv_debug_check_guards": (I32, [C.POINTER(I32)]),
    "gnnv_row_stride": (I32, [I32]),
    "gnnv_launch_count": (U64, []),
    "gnnv_graph_load": (I32, [VP, VP, I64, I64, VP, I32, I32, VP, I32, I32, PP]),
    "gnnv_graph_free": (I32, [VP]),
    "gnnv_graph_info": (I32, [VP, C.POINTER(GraphView)]),
    "gnnv_comm_unique_id": (I32, [VP]),
    "gnnv_comm_init": (I32, [I32, I32, VP, I32, PP]),
    "gnnv_comm_free": (I32, [VP]),
    "gnnv_allreduce_sum": (I32, [VP, VP, I64, VP]),
    "gnnv_cache_build": (I32, [VP, F64, I32, I32, VP, I32, PP]),
    "gnnv_cache_ipc_handle": (I32, [VP, VP]),
    "gnnv_cache_update": (I32, [VP, VP, VP, VP]),
    "gnnv_cache_counters": (I32, [VP, VP]),
    "gnnv_cache_owners": (I32, [VP, PP]),
    "gnnv_cache_open_peers": (I32, [VP, VP]),
    "gnnv_cache_free": (I32, [VP]),
    "gnnv_cache_info": (I32, [VP, C.POINTER(CacheView)]),
    "gnnv_blocks_create": (I32, [VP, I32, VP, I32, PP]),
    "gnnv_blocks_free": (I32, [VP]),
    "gnnv_sample": (I32, [VP, VP, I32, VP, I32, U64, VP, VP]),
    "gnnv_blocks_info": (I32, [VP, I32, VP, C.POINTER(BlockView)]),
    "gnnv_blocks_device_sizes": (VP, [VP]),
    "gnnv_blocks_num_layers": (I32, [VP]),
    "gnnv_gather": (I32, [VP, VP, VP, VP, VP]),
    "gnnv_layer_fwd": (I32, [VP, I32, C.POINTER(LayerDesc), VP, VP, VP, VP, VP, VP]),
    "gnnv_layer_bwd": (I32, [VP, I32, C.POINTER(LayerDesc), VP, VP, VP, VP, VP, VP, VP, VP, VP]),
    "gnnv_ce_loss": (I32, [VP, VP, VP, I32, I32, I32, VP, VP, VP]),
    "gnnv_sgd": (I32, [VP, VP, I64, F32, VP]),
    "gnnv_dense_fwd": (I32, [VP, I32, VP, I32, I32, VP, VP, VP, I32, I32, I64, I32, I32, VP]),
    "gnnv_dense_dx": (I32, [VP, I32, I32, VP, I32, VP, I32, VP, I32, I64, I32, VP]),
    "gnnv_dense_dw": (I32, [VP, I32, VP, I32, I32, VP, I32, I32, I64, VP, VP, I32, VP]),
    "gnnv_trainer_create": (I32, [VP, VP, C.POINTER(ModelDesc), VP, VP, PP]),
    "gnnv_trainer_free": (I32, [VP]),
    "gnnv_trainer_num_params": (I64, [VP]),
    "gnnv_trainer_get": (I32, [VP, VP, VP]),
    "gnnv_trainer_set_params": (I32, [VP, VP]),
    "gnnv_trainer_blocks": (VP, [VP]),
    "gnnv_trainer_x_level": (I32, [VP]),
    "gnnv_trainer_rowidx": (I32, [VP, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "gnnv_trainer_loss_async": (I32, [VP, VP, VP]),
    "gnnv_trainer_loss_result": (I32, [VP, C.c_int64, VP]),
    "gnnv_trainer_set_locality": (I32, [VP, F64]),
    "gnnv_blocks_set_locality": (I32, [VP, VP, F64]),
    "gnnv_trainer_activation": (I32, [VP, I32, PP, C.POINTER(I32)]),
    "gnnv_trainer_aggregate": (I32, [VP, I32, PP, C.POINTER(I32)]),
    "gnnv_trainer_relu_bits": (I32, [VP, I32, PP, C.POINTER(I32)]),
    "gnnv_trainer_l2push": (I32, [VP]),
    "gnnv_trainer_bf16act": (I32, [VP]),
    "gnnv_trainer_table16": (I32, [VP]),
    "gnnv_trainer_activation16": (I32, [VP, I32, PP, C.POINTER(I32)]),
    "gnnv_trainer_gradient16": (I32, [VP, I32, PP, C.POINTER(I32)]),
    "gnnv_trainer_dw16": (I32, [VP]),
    "gnnv_trainer_fwd16": (I32, [VP]),
    "gnnv_trainer_tail16": (I32, [VP]),
    "gnnv_trainer_last_rows": (I32, [VP]),
    "gnnv_host_read_probe": (I32, [VP, I64, I32, C.POINTER(C.c_float), VP]),
    "gnnv_trainer_aggregate16": (I32, [VP, I32, PP, C.POINTER(I32)]),
    "gnnv_trainer_dw16_operands": (I32, [VP, PP, PP, C.POINTER(I32)]),
    "gnnv_step": (I32, [VP, VP, I32, I32, I32, U64, F32, C.POINTER(F32), C.POINTER(StepTiming), VP]),
    "gnnv_trainer_stats": (I32, [VP, VP]),
    "gnnv_trainer_prefetch": (I32, [VP, VP, I32, I32, U64, VP]),
    "gnnv_trainer_join_prefetch": (I32, [VP, VP]),
    "gnnv_trainer_read_loss": (I32, [VP, C.POINTER(F32), VP]),
    "gnnv_trainer_timeline": (I32, [VP, I32]),
    "gnnv_trainer_timeline_read": (I32, [VP, C.POINTER(Segment), I32, C.POINTER(I32)]),
}
EXPORTS = sorted(_SIGS)

_lib: Optional[C.CDLL] = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libgnnv.so (raises if it is missing -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libgnnv.so not built at {path}: run `python -m paper_2404_09544_b200.build`")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(st: int):
    if st != OK:
        raise GnnvError(st, load().gnnv_last_error().decode(errors="replace"))


def ptr(x) -> Optional[int]:
    """Device/host pointer of a torch tensor, numpy array, int or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def stream_ptr(s=None) -> Optional[int]:
    if s is None:
        import torch
        s = torch.cuda.current_stream()
    if isinstance(s, int):
        return s
    return s.cuda_stream


def version() -> str:
    return load().gnnv_version().decode()


def set_option(name: str, value: int):
    """gnnv_set_option: opt-in variant switches (1 on, 0 off, -1 environment)."""
    _check(load().gnnv_set_option(name.encode(), int(value)))


def check_guards() -> str:
    """gnnv_debug_check_guards: '' if no guard region changed, else the report."""
    n = C.c_int32(0)
    _check(load().gnnv_debug_check_guards(C.byref(n)))
    return load().gnnv_last_error().decode(errors="replace") if n.value else ""


def launch_count() -> int:
    return int(load().gnnv_launch_count())


def host_read_probe(h_ptr: int, nbytes: int, reps: int = 5, stream: int = 0) -> float:
    """Device ms of `reps` SM zero-copy read passes over pinned host memory."""
    ms = C.c_float(0.0)
    _check(load().gnnv_host_read_probe(C.c_void_p(h_ptr), nbytes, reps, C.byref(ms), C.c_void_p(stream)))
    return float(ms.value)


def row_stride(d: int) -> int:
    return int(load().gnnv_row_stride(d))


def preload_nccl():
    """Make libnccl.so.2 (the torch-bundled one) resolvable for dlopen."""
    try:
        import nvidia.nccl  # type: ignore
        for p in nvidia.nccl.__path__:
            cand = os.path.join(p, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                C.CDLL(cand, mode=C.RTLD_GLOBAL)
                os.environ.setdefault("GNNV_NCCL_LIB", cand)
                return cand
    except Exception:
        pass
    return None


# --------------------------------------------------------------- handles
class Graph:
    """gnnv_graph_load.  Keeps the borrowed host arrays alive."""

    def __init__(self, indptr, indices, feats: np.ndarray, d: int, labels, n_classes: int, device: int = 0):
        lib = load()
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int32)
        if not (feats.flags.c_contiguous and feats.dtype == np.float32 and feats.ctypes.data % 16 == 0):
            raise ValueError("feats must be C-contiguous float32, 16-byte aligned")
        self.feats = feats
        self.labels = np.ascontiguousarray(labels, dtype=np.int32)
        self.n = int(self.indptr.shape[0] - 1)
        self.d = int(d)
        self.stride = int(feats.shape[1])
        self.n_classes = int(n_classes)
        h = C.c_void_p()
        _check(lib.gnnv_graph_load(ptr(self.indptr), ptr(self.indices), self.n, int(self.indices.shape[0]),
                                   ptr(feats), self.d, self.stride, ptr(self.labels), self.n_classes, device,
                                   C.byref(h)))
        self.h = h

    @classmethod
    def from_data(cls, gd, device: int = 0):
        return cls(gd.indptr, gd.indices, gd.feats, gd.d, gd.labels, gd.C, device)

    def info(self) -> GraphView:
        v = GraphView()
        _check(load().gnnv_graph_info(self.h, C.byref(v)))
        return v

    def free(self):
        if getattr(self, "h", None):
            load().gnnv_graph_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Comm:
    def __init__(self, rank: int, world: int, unique_id: Optional[bytes], device: int):
        """unique_id None: a host-only comm (no NCCL; see gnnv_comm_init)."""
        h = C.c_void_p()
        if unique_id is None:
            buf = None
        else:
            preload_nccl()
            buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(load().gnnv_comm_init(rank, world, buf, device, C.byref(h)))
        self.h, self.rank, self.world = h, rank, world

    @staticmethod
    def unique_id() -> bytes:
        preload_nccl()
        buf = C.create_string_buffer(128)
        _check(load().gnnv_comm_unique_id(buf))
        return buf.raw

    def allreduce_sum(self, t, stream=None):
        _check(load().gnnv_allreduce_sum(self.h, ptr(t), int(t.numel()), stream_ptr(stream)))

    def free(self):
        if getattr(self, "h", None):
            load().gnnv_comm_free(self.h)
            self.h = None


class Cache:
    def __init__(self, g: Graph, ratio: float, policy: int = POLICY_DEGREE, placement: int = PLACE_REPLICA,
                 comm: Optional[Comm] = None, virtual_shards: int = 1):
        h = C.c_void_p()
        _check(load().gnnv_cache_build(g.h, float(ratio), policy, placement, comm.h if comm else None,
                                       virtual_shards, C.byref(h)))
        self.h, self.g = h, g

    def info(self) -> CacheView:
        v = CacheView()
        _check(load().gnnv_cache_info(self.h, C.byref(v)))
        return v

    def update(self, blocks: "Blocks", X, stream=None):
        """Dynamic cache: admit the misses of the batch gathered into X."""
        _check(load().gnnv_cache_update(self.h, blocks.h, ptr(X), stream_ptr(stream)))

    def counters(self) -> np.ndarray:
        """Dynamic cache: cumulative (hits, misses, replaced, admitted)."""
        out = np.zeros(4, np.int64)
        _check(load().gnnv_cache_counters(self.h, ptr(out)))
        return out

    def owners_ptr(self) -> int:
        p = C.c_void_p()
        _check(load().gnnv_cache_owners(self.h, C.byref(p)))
        return int(p.value)

    def ipc_handle(self) -> bytes:
        """SHARDED: this rank's 64-byte CUDA IPC handle of its shard."""
        buf = C.create_string_buffer(64)
        _check(load().gnnv_cache_ipc_handle(self.h, buf))
        return buf.raw

    def open_peers(self, handles: Sequence[bytes]):
        """SHARDED with a host-only comm: map the other ranks' shards."""
        blob = b"".join(bytes(h) for h in handles)
        _check(load().gnnv_cache_open_peers(self.h, C.create_string_buffer(blob, len(blob))))

    def free(self):
        if getattr(self, "h", None):
            load().gnnv_cache_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _i32arr(xs: Sequence[int]):
    a = (C.c_int32 * max(1, len(xs)))()
    for i, x in enumerate(xs):
        a[i] = int(x)
    return a


class Blocks:
    def __init__(self, g: Graph, max_seeds: int, fanouts: Sequence[int], h: Optional[C.c_void_p] = None):
        self.g, self.fanouts, self.L = g, list(fanouts), len(fanouts)
        self.owned = h is None
        if h is None:
            h = C.c_void_p()
            _check(load().gnnv_blocks_create(g.h, max_seeds, _i32arr(fanouts), len(fanouts), C.byref(h)))
        self.h = h

    def sample(self, d_seeds, n_seeds: int, rng_seed: int, stream=None):
        _check(load().gnnv_sample(self.g.h, ptr(d_seeds), int(n_seeds), _i32arr(self.fanouts), self.L,
                                  int(rng_seed) & 0xFFFFFFFFFFFFFFFF, self.h, stream_ptr(stream)))

    def set_locality(self, cache: Optional["Cache"], bias: float):
        """Locality-biased sampling (NEXT-2): cached neighbours weigh 1 + 4 bias."""
        _check(load().gnnv_blocks_set_locality(self.h, cache.h if cache else None, float(bias)))

    def info(self, sync: bool = True, stream=None) -> List[BlockView]:
        arr = (BlockView * self.L)()
        _check(load().gnnv_blocks_info(self.h, 1 if sync else 0, stream_ptr(stream), arr))
        return [arr[i] for i in range(self.L)]

    def device_sizes(self) -> int:
        return int(load().gnnv_blocks_device_sizes(self.h))

    def free(self):
        if self.owned and getattr(self, "h", None):
            load().gnnv_blocks_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def gather(cache: Cache, blocks: Blocks, X, stats=None, stream=None):
    _check(load().gnnv_gather(cache.h, blocks.h, ptr(X), ptr(stats), stream_ptr(stream)))


def layer_desc(d_in, d_out, in_stride, kind=KIND_SAGE, aggr=AGGR_MEAN, act=ACT_RELU, prec=PREC_FP32) -> LayerDesc:
    return LayerDesc(int(d_in), int(d_out), int(in_stride), int(kind), int(aggr), int(act), int(prec))


def layer_fwd(blocks: Blocks, layer: int, ld: LayerDesc, Hsrc, W, b, Hdst, saveA, stream=None):
    _check(load().gnnv_layer_fwd(blocks.h, layer, C.byref(ld), ptr(Hsrc), ptr(W), ptr(b), ptr(Hdst), ptr(saveA),
                                 stream_ptr(stream)))


def layer_bwd(blocks: Blocks, layer: int, ld: LayerDesc, Gdst, Hdst, Hsrc, saveA, W, Gsrc, dW, db, stream=None):
    _check(load().gnnv_layer_bwd(blocks.h, layer, C.byref(ld), ptr(Gdst), ptr(Hdst), ptr(Hsrc), ptr(saveA), ptr(W),
                                 ptr(Gsrc), ptr(dW), ptr(db), stream_ptr(stream)))


def ce_loss(blocks: Blocks, g: Graph, logits, n_classes, stride, n_global, loss, dlogits, stream=None):
    _check(load().gnnv_ce_loss(blocks.h, g.h, ptr(logits), int(n_classes), int(stride), int(n_global), ptr(loss),
                               ptr(dlogits), stream_ptr(stream)))


def dense_fwd(X1, ld1, X2, ld2, K1, W, b, Y, ldy, N, M, relu=True, prec=PREC_TF32, stream=None):
    _check(load().gnnv_dense_fwd(ptr(X1), ld1, ptr(X2), ld2, K1, ptr(W), ptr(b), ptr(Y), ldy, N, int(M),
                                 1 if relu else 0, prec, stream_ptr(stream)))


def dense_dx(G, ldg, N, W, K1, Y1, ld1, Y2, ld2, M, prec=PREC_TF32, stream=None):
    _check(load().gnnv_dense_dx(ptr(G), ldg, N, ptr(W), K1, ptr(Y1), ld1, ptr(Y2), ld2, int(M), prec,
                                stream_ptr(stream)))


def dense_dw(X1, ld1, X2, ld2, K1, G, ldg, N, M, dW, db=None, prec=PREC_TF32, stream=None):
    _check(load().gnnv_dense_dw(ptr(X1), ld1, ptr(X2), ld2, K1, ptr(G), ldg, N, int(M), ptr(dW), ptr(db), prec,
                                stream_ptr(stream)))


def sgd(params, grads, n: int, lr: float, stream=None):
    _check(load().gnnv_sgd(ptr(params), ptr(grads), int(n), float(lr), stream_ptr(stream)))


def flat_params(weights) -> np.ndarray:
    """[(W, b), ...] -> the trainer's flat layout (W row-major, then b, per layer)."""
    return np.concatenate([np.concatenate([np.asarray(W, np.float32).ravel(), np.asarray(b, np.float32).ravel()])
                           for W, b in weights]).astype(np.float32)


def unflat_params(flat: np.ndarray, dims: Sequence[int], kind: int = KIND_SAGE):
    out, off = [], 0
    for i in range(len(dims) - 1):
        rows = (2 if kind == KIND_SAGE else 1) * dims[i]
        W = flat[off: off + rows * dims[i + 1]].reshape(rows, dims[i + 1])
        off += rows * dims[i + 1]
        b = flat[off: off + dims[i + 1]]
        off += dims[i + 1]
        out.append((W, b))
    return out


class Trainer:
    """gnnv_trainer_*: whole-iteration runner (gnnv_step)."""

    def __init__(self, g: Graph, cache: Cache, dims: Sequence[int], fanouts: Sequence[int], max_seeds: int,
                 weights, kind=KIND_SAGE, aggr=AGGR_MEAN, prec=PREC_FP32, comm: Optional[Comm] = None):
        md = ModelDesc()
        md.L = len(fanouts)
        for i, x in enumerate(dims):
            md.dims[i] = int(x)
        for i, x in enumerate(fanouts):
            md.fanouts[i] = int(x)
        md.max_seeds, md.kind, md.aggr, md.prec = int(max_seeds), int(kind), int(aggr), int(prec)
        self.dims, self.kind, self.L = list(dims), kind, len(fanouts)
        flat = flat_params(weights)
        h = C.c_void_p()
        _check(load().gnnv_trainer_create(g.h, cache.h, C.byref(md), ptr(flat), comm.h if comm else None,
                                          C.byref(h)))
        self.h, self.g, self.cache, self.comm = h, g, cache, comm
        self.nparams = int(load().gnnv_trainer_num_params(h))
        self._max_seeds, self._fanouts = max_seeds, list(fanouts)

    @property
    def blocks(self) -> "Blocks":
        """The blocks of the last step (borrowed; with the Eq.4 prefetch the
        trainer alternates between two buffer sets)."""
        b = Blocks(self.g, self._max_seeds, self._fanouts, h=C.c_void_p(load().gnnv_trainer_blocks(self.h)))
        # the last hop's indices are cache-table rows (gnnv_trainer_last_rows):
        # the cache's degree order maps them back to vertex ids
        b.last_rows_order = self.cache.info().d_order if self.last_rows() else None
        return b

    def step(self, seeds, n_seeds: int, n_global: int, rng_seed: int, lr: float, on_host: bool = True,
             want_loss: bool = True, timing: bool = False, stream=None):
        loss = C.c_float(0.0)
        tm = StepTiming()
        if on_host:
            seeds = np.ascontiguousarray(seeds, dtype=np.int32)
        _check(load().gnnv_step(self.h, ptr(seeds), int(n_seeds), 1 if on_host else 0, int(n_global),
                                int(rng_seed) & 0xFFFFFFFFFFFFFFFF, float(lr),
                                C.byref(loss) if want_loss else None, C.byref(tm) if timing else None,
                                stream_ptr(stream)))
        return (float(loss.value) if want_loss else None), (tm.as_dict() if timing else None)

    def prefetch(self, seeds, n_seeds: int, rng_seed: int, on_host: bool = True, stream=None):
        """Sample + gather the next step's batch on the side stream (Eq.4 overlap)."""
        if on_host:
            seeds = np.ascontiguousarray(seeds, dtype=np.int32)
        _check(load().gnnv_trainer_prefetch(self.h, ptr(seeds), int(n_seeds), 1 if on_host else 0,
                                            int(rng_seed) & 0xFFFFFFFFFFFFFFFF, stream_ptr(stream)))

    def join_prefetch(self, stream=None):
        """`stream` waits for the pending prefetch (not consumed)."""
        _check(load().gnnv_trainer_join_prefetch(self.h, stream_ptr(stream)))

    def read_loss(self, stream=None) -> float:
        out = C.c_float(0.0)
        _check(load().gnnv_trainer_read_loss(self.h, C.byref(out), stream_ptr(stream)))
        return float(out.value)

    def loss_async(self, stream=None) -> int:
        """Enqueue the last step's loss read-back; returns a ticket."""
        t = C.c_int64(0)
        _check(load().gnnv_trainer_loss_async(self.h, C.byref(t), stream_ptr(stream)))
        return int(t.value)

    def loss_result(self, ticket: int) -> float:
        out = C.c_float(0.0)
        _check(load().gnnv_trainer_loss_result(self.h, int(ticket), C.byref(out)))
        return float(out.value)

    def params(self) -> np.ndarray:
        out = np.empty(self.nparams, np.float32)
        _check(load().gnnv_trainer_get(self.h, ptr(out), None))
        return out

    def grads(self) -> np.ndarray:
        out = np.empty(self.nparams, np.float32)
        _check(load().gnnv_trainer_get(self.h, None, ptr(out)))
        return out

    def set_params(self, flat: np.ndarray):
        flat = np.ascontiguousarray(flat, np.float32)
        _check(load().gnnv_trainer_set_params(self.h, ptr(flat)))

    def set_locality(self, bias: float):
        """Locality-biased sampling (NEXT-2) for the trainer's batches."""
        _check(load().gnnv_trainer_set_locality(self.h, float(bias)))

    def x_level(self) -> int:
        """Frontier level whose rows X holds: L (all of F_L), L-1 (dst prefix) or -1 (none)."""
        return int(load().gnnv_trainer_x_level(self.h))

    def rowidx(self):
        """(device ptr of int32[n_L] cache rows of F_L, device ptr of the table) or (None, None)."""
        r, t = C.c_void_p(), C.c_void_p()
        _check(load().gnnv_trainer_rowidx(self.h, C.byref(r), C.byref(t)))
        return r.value, t.value

    def activation(self, i: int):
        p = C.c_void_p()
        st = C.c_int32()
        _check(load().gnnv_trainer_activation(self.h, i, C.byref(p), C.byref(st)))
        return int(p.value or 0), int(st.value)

    def aggregate(self, i: int):
        """(device pointer, stride) of layer i's aggregate A^i of the last step."""
        p = C.c_void_p()
        st = C.c_int32()
        _check(load().gnnv_trainer_aggregate(self.h, i, C.byref(p), C.byref(st)))
        return int(p.value or 0), int(st.value)

    def relu_bits(self, i: int):
        """(device pointer, words per row) of layer i's ReLU bits (TF32), or (0, 0)."""
        p = C.c_void_p()
        w = C.c_int32()
        _check(load().gnnv_trainer_relu_bits(self.h, i, C.byref(p), C.byref(w)))
        return int(p.value or 0), int(w.value)

    def l2push(self) -> bool:
        return bool(load().gnnv_trainer_l2push(self.h))

    def bf16act(self) -> bool:
        return bool(load().gnnv_trainer_bf16act(self.h))

    def table16(self) -> bool:
        return bool(load().gnnv_trainer_table16(self.h))

    def activation16(self, i: int):
        """(device pointer, row stride) of the bf16 copy of H^i, or (0, 0)."""
        p = C.c_void_p()
        ld = C.c_int32()
        _check(load().gnnv_trainer_activation16(self.h, i, C.byref(p), C.byref(ld)))
        return int(p.value or 0), int(ld.value)

    def gradient16(self, i: int):
        """(device pointer, row stride) of the bf16 dL/dH^i layer i's dW read, or (0, 0)."""
        p = C.c_void_p()
        ld = C.c_int32()
        _check(load().gnnv_trainer_gradient16(self.h, i, C.byref(p), C.byref(ld)))
        return int(p.value or 0), int(ld.value)

    def dw16(self) -> bool:
        return bool(load().gnnv_trainer_dw16(self.h))

    def fwd16(self) -> bool:
        return bool(load().gnnv_trainer_fwd16(self.h))

    def tail16(self) -> bool:
        return bool(load().gnnv_trainer_tail16(self.h))

    def last_rows(self) -> bool:
        return bool(load().gnnv_trainer_last_rows(self.h))

    def aggregate16(self, i: int):
        """(device pointer, row stride) of the bf16 copy of A^i the kind::f16 GEMMs read, or (0, 0)."""
        p = C.c_void_p()
        ld = C.c_int32()
        _check(load().gnnv_trainer_aggregate16(self.h, i, C.byref(p), C.byref(ld)))
        return int(p.value or 0), int(ld.value)

    def dw16_operands(self):
        """(X16, A16, row stride): layer 1's bf16 dW operands of the last step."""
        x = C.c_void_p()
        a = C.c_void_p()
        ld = C.c_int32()
        _check(load().gnnv_trainer_dw16_operands(self.h, C.byref(x), C.byref(a), C.byref(ld)))
        return int(x.value or 0), int(a.value or 0), int(ld.value)

    def timeline(self, on: bool):
        _check(load().gnnv_trainer_timeline(self.h, 1 if on else 0))

    def timeline_read(self):
        """{name: (total_ms, count)} since the last read (synchronises)."""
        arr = (Segment * 256)()
        n = C.c_int32()
        _check(load().gnnv_trainer_timeline_read(self.h, arr, 256, C.byref(n)))
        return {arr[i].name.decode(): (float(arr[i].total_ms), int(arr[i].count)) for i in range(min(n.value, 256))}

    def stats(self) -> np.ndarray:
        out = np.zeros(4, np.int64)
        _check(load().gnnv_trainer_stats(self.h, ptr(out)))
        return out

    def free(self):
        if getattr(self, "h", None):
            load().gnnv_trainer_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
