"""-m gpu: pins the oracle's Philox draw layout to the library routine.

oracle/philox.py:draw claims draw(seed, h, v, s) equals
curand_init(seed, (h << 32) | v, s, &st); curand(&st) with cuRAND's
Philox4_32_10 -- i.e. word s & 3 of Philox4x32-10(ctr = (s >> 2, 0, v, h),
key = seed).  The CPU pins (tests/golden/philox_kat.txt) fix the block
function; this fixes the counter/key layout against an implementation this
repo did not write (tests/native/curand_probe.cu, built here with nvcc).
Reading Q4; the RNG is the paper's open choice (Eq.2,
P:240-244).
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest
import torch

from oracle.philox import draw

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def probe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("curand") / "libcurand_probe.so")
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared", "-Xcompiler", "-fPIC",
                    os.path.join(HERE, "native", "curand_probe.cu"), "-o", out], check=True)
    torch.cuda.init()
    lib = ctypes.CDLL(out)
    lib.curand_probe_draws.argtypes = [ctypes.c_uint64] + [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_void_p]
    return lib


def curand_draws(lib, seed, h, v, s):
    h, v, s = (np.ascontiguousarray(x, dtype=np.uint32) for x in (h, v, s))
    out = np.zeros(h.size, dtype=np.uint32)
    assert lib.curand_probe_draws(seed, h.ctypes.data, v.ctypes.data, s.ctypes.data, h.size, out.ctypes.data) == 0
    return out


@pytest.mark.parametrize("seed", [0, 0x5EED, 0x5EED + 10, 0x123456789ABCDEF0, 2**64 - 1])
def test_draw_equals_curand_philox(probe, seed):
    rng = np.random.default_rng(seed & 0xFFFF)
    n = 4096
    h = rng.integers(0, 8, n)
    v = np.concatenate([rng.integers(0, 2**31 - 1, n - 4), [0, 1, 2**31 - 2, 111059955]])
    s = rng.integers(0, 32, n)  # every draw index a fanout <= 32 uses, all four words
    got = curand_draws(probe, seed, h, v, s)
    want = draw(seed, h, v, s).astype(np.uint32)
    np.testing.assert_array_equal(got, want)


def test_draw_grid_equals_curand(probe):
    # every (h, s) for a few nodes: all counter words and offsets 0..31
    h, v, s = np.meshgrid(np.arange(4), np.array([0, 5, 2449028]), np.arange(32), indexing="ij")
    got = curand_draws(probe, 0x5EED, h.ravel(), v.ravel(), s.ravel())
    np.testing.assert_array_equal(got, draw(0x5EED, h.ravel(), v.ravel(), s.ravel()).astype(np.uint32))
