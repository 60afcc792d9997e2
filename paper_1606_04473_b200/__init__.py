"""B200-native Aggregate Risk Analysis (arxiv 1606.04473 hot path).

The product is ``libara.so`` (C ABI, include/ara.h) — hand-written sm_100a
kernels for ELT densification, the ARA trial loop and device PML/TVaR, plus a
C++ host runtime (chunked H2D, NCCL YLT all-gather).  ``ara`` is the ctypes
binding with the same names.
"""
from .ara import *  # noqa: F401,F403
from .ara import Context, AraError  # noqa: F401
