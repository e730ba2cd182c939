"""B200-native HybridQ state-vector core (arXiv 2111.06868).

The product is the C-ABI library ``lib/libhq.so`` (header ``include/hq.h``):
hand-written sm_100a kernels that apply dense, fused k-qubit gates to a 2^n
amplitude vector, a host fusion planner and a distributed qubit-remap layer
(NCCL).  ``hq`` is a thin ctypes binding with the same function names.
"""
from . import hq  # noqa: F401
from .hq import *  # noqa: F401,F403

__version__ = "0.1.0"
