"""Build libgnnv.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2404_09544_b200.build [--force] [--debug]
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libgnnv.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    cands = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl", "include"))
    try:
        import nvidia.nccl  # type: ignore

        cands = [os.path.join(p, "include") for p in nvidia.nccl.__path__] + cands
    except Exception:
        pass
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")


def _cudart_dirs():
    """libcudart.so.12 the process (torch) already uses comes first."""
    dirs = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "cuda_runtime", "lib"))
    return dirs + ["/usr/local/cuda/lib64"]


def _flags(debug: bool):
    f = ARCH + ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                "-I" + os.path.join(ROOT, "include"), "-I" + _nccl_include(), "-Xptxas", "-v"]
    if debug:
        f += ["-G"]
    return f


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _digest(debug: bool) -> str:
    h = hashlib.sha256()
    for p in _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "gnnv.h")]:
        h.update(os.path.relpath(p, ROOT).encode())
        h.update(open(p, "rb").read())
    h.update(" ".join(f for f in _flags(debug) if not f.startswith("-I")).encode())
    return h.hexdigest()


def build(force: bool = False, debug: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    stamp = os.path.join(BUILD, "stamp")
    dig = _digest(debug)
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == dig:
        return LIB
    flags = _flags(debug)

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [NVCC] + flags + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        log = os.path.join(BUILD, os.path.basename(src) + ".ptxas.txt")
        with open(log, "w") as fh:
            fh.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = LIB + ".tmp"
    rpath = ":".join(_cudart_dirs())
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "-cudart", "shared", "-Xlinker", "-rpath=" + rpath]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as fh:
        fh.write(dig)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, debug="--debug" in sys.argv, verbose=True)
