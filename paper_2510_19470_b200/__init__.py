"""B200-native HybridEP MoE-layer hot path.

The compute path is libhep.so (C++ host + sm_100a CUDA kernels + NCCL), reached
through the C-ABI in include/hep.h.  `_lib` fails loudly when the library is
missing; there is no CPU fallback.
"""
import os as _os

# The step runs on several streams per GPU (main, dispatch side stream, expert
# All-Gather stream, H2D/D2H) with cross-GPU flag waits on them.  With CUDA's default
# 8 hardware work queues, unrelated streams can share a queue and inherit false
# ordering, which can close a wait cycle across GPUs; give every stream its own queue.
# Must be set before the CUDA context exists (import this package first, or export it).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from ._lib import (DomainError, HepError, InvalidArgument, NcclError, RuntimeFailure,  # noqa: F401
                   CudaError, declared_symbols, lib)
from . import topology  # noqa: F401

__all__ = ["topology", "lib", "HepError", "DomainError", "InvalidArgument", "RuntimeFailure"]
