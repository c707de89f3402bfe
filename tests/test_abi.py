"""CPU checks of the C-ABI boundary: libgnnv.so builds, loads, and exports
every symbol include/gnnv.h declares; the binding covers them; host-side
parameter validation works without a GPU (no compute calls)."""
import os
import re
import subprocess

import pytest

from paper_2404_09544_b200 import gnnv
from paper_2404_09544_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gnnv.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gnnv_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    build()
    return gnnv.load()


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ["gnnv_graph_load", "gnnv_cache_build", "gnnv_sample", "gnnv_gather", "gnnv_layer_fwd",
                 "gnnv_layer_bwd", "gnnv_step"]:
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", gnnv.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(gnnv_[a-z0-9_]+)\b", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_binding_covers_every_declared_symbol(lib):
    assert sorted(declared_symbols()) == gnnv.EXPORTS


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gnnv.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_side_errors_without_gpu(lib):
    assert gnnv.version().startswith("0.")
    assert gnnv.row_stride(1433) == 1436 and gnnv.row_stride(100) == 100 and gnnv.row_stride(47) == 48
    import ctypes as C
    h = C.c_void_p()
    # null pointers -> parameter error before any CUDA call
    st = lib.gnnv_graph_load(None, None, 10, 0, None, 4, 4, None, 2, 0, C.byref(h))
    assert st == gnnv.ERR_PARAM
    assert b"null" in lib.gnnv_last_error()
    assert lib.gnnv_cache_build(None, 0.5, 1, 0, None, 1, C.byref(h)) == gnnv.ERR_PARAM
    assert lib.gnnv_blocks_create(None, 1, None, 1, C.byref(h)) == gnnv.ERR_PARAM
    assert lib.gnnv_sgd(None, None, 1, 0.1, None) == gnnv.ERR_PARAM
