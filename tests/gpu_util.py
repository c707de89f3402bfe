"""Helpers for the -m gpu parity tests (CUDA path vs oracle)."""
import ctypes

import numpy as np
import torch

from paper_2404_09544_b200 import gnnv
from paper_2404_09544_b200.build import build

_built = False


def lib():
    global _built
    if not _built:
        build()
        _built = True
    return gnnv.load()


def dev_i32(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def dev_f32(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def read_i32(p, n):
    """Copy n int32 from a raw device pointer."""
    out = torch.empty(int(n), dtype=torch.int32, device="cuda")
    if n:
        torch.cuda.synchronize()
        res = _cudart().cudaMemcpy(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(int(p)),
                                   ctypes.c_size_t(int(n) * 4), 3)  # cudaMemcpyDeviceToDevice
        assert int(res) == 0, res
    return out.cpu().numpy()


def read_f32(p, rows, stride):
    """Copy a [rows x stride] fp32 matrix from a raw device pointer."""
    out = torch.empty((int(rows), int(stride)), dtype=torch.float32, device="cuda")
    if rows:
        torch.cuda.synchronize()
        res = _cudart().cudaMemcpy(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(int(p)),
                                   ctypes.c_size_t(int(rows) * int(stride) * 4), 3)
        assert int(res) == 0, res
    return out.cpu().numpy()


_rt = None


def _cudart():
    global _rt
    if _rt is None:
        _rt = ctypes.CDLL("libcudart.so.12")
    return _rt


def blocks_to_host(blocks: gnnv.Blocks):
    """Per hop: (n_dst, n_src, indptr, indices, src_global) on the host."""
    torch.cuda.synchronize()
    views = blocks.info(sync=True)
    out = []
    for v in views:
        indptr = read_i32(v.d_indptr, v.n_dst + 1)
        indices = read_i32(v.d_indices, v.nnz)
        F = read_i32(v.d_src_global, v.n_src)
        out.append((int(v.n_dst), int(v.n_src), indptr, indices, F))
    return out


def assert_close_cond(got, ref, mag, rtol, what=""):
    """Condition-aware elementwise bound (reading Q17):
    |got - ref| <= rtol * mag + 1e-30, mag = the same expression on |.|."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    mag = np.asarray(mag, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    err = np.abs(got - ref)
    bound = rtol * mag + 1e-30
    bad = err > bound
    if bad.any():
        i = np.unravel_index(np.argmax(err / bound), err.shape)
        raise AssertionError(f"{what}: {int(bad.sum())} of {err.size} elements exceed rtol={rtol}; worst at {i}: "
                             f"got {got[i]!r} ref {ref[i]!r} mag {mag[i]!r}")


def normwise(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))
