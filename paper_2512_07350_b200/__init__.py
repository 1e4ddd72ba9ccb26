"""B200-native Latent Parallelism (LP) engine — arXiv 2512.07350.

The product is liblp_b200.so (C-ABI in include/lp_b200.h: hand-written sm_100a
kernels + the C++ step loop + NCCL); ``lp`` is its Python face, mirroring the
reference's python module (lpsim).
"""
from . import lp  # noqa: F401
from ._lib import LpError, lib  # noqa: F401

__version__ = "0.1.0"
