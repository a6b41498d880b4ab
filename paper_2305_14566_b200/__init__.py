"""B200-native slide-wise Omni-Seg prediction (arxiv 2305.14566).

The product is libomniseg.so (C ABI, include/omniseg.h) built from csrc/ for
sm_100a; this package is its thin Python binding (lib.py) plus the in-tree
build (build.py). No CPU fallback: without the CUDA library every call raises.
"""
from .lib import Omniseg, OmnisegError, band_rows, load  # noqa: F401
