"""Probe: can a /dev/shm memmap be page-locked in place (cudaHostRegister)?"""
import ctypes
import mmap
import os

import numpy as np

rt = ctypes.CDLL("libcudart.so.12")
rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
rt.cudaHostUnregister.argtypes = [ctypes.c_void_p]
rt.cudaGetErrorString.restype = ctypes.c_char_p
rt.cudaFree(None)
path = "/dev/shm/gnnv_probe.npy"
np.save(path, np.ones((1 << 20, 100), np.float32))
MAPPED, PORTABLE, RO = 2, 1, 8
for mode in ("r", "r+", "c"):
    a = np.load(path, mmap_mode=mode)
    for name, flags in (("mapped|portable|ro", MAPPED | PORTABLE | RO), ("mapped|portable", MAPPED | PORTABLE)):
        rc = rt.cudaHostRegister(a.ctypes.data, a.nbytes, flags)
        print(mode, name, rc, rt.cudaGetErrorString(rc).decode(), flush=True)
        rt.cudaGetLastError()
        if rc == 0:
            rt.cudaHostUnregister(a.ctypes.data)
    # page-aligned base of the same mapping
    base = a.ctypes.data & ~4095
    rc = rt.cudaHostRegister(base, a.nbytes + (a.ctypes.data - base), MAPPED | PORTABLE | RO)
    print(mode, "aligned ro", rc, rt.cudaGetErrorString(rc).decode(), flush=True)
    rt.cudaGetLastError()
    if rc == 0:
        rt.cudaHostUnregister(base)
    del a
fd = os.open(path, os.O_RDONLY)
m = mmap.mmap(fd, 0, mmap.MAP_SHARED, mmap.PROT_READ)
buf = (ctypes.c_char * len(m)).from_buffer_copy(b"") if False else None
os.close(fd)
os.remove(path)
