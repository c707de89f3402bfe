"""B200-native hot path of GNNavigator (arXiv 2404.09544): sampled
GraphSAGE/GCN mini-batch iteration behind the libgnnv C-ABI.

The compute lives in libgnnv.so (hand-written CUDA for sm_100a, see
csrc/); `gnnv` is the thin ctypes binding.  Importing the package does not
require a GPU; calling into it requires the built library.
"""
from . import gnnv  # noqa: F401

__all__ = ["gnnv"]
