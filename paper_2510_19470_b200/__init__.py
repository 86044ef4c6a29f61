"""B200-native HybridEP MoE-layer hot path.

The compute path is libhep.so (C++ host + sm_100a CUDA kernels + NCCL), reached
through the C-ABI in include/hep.h.  `_lib` fails loudly when the library is
missing; there is no CPU fallback.
"""
from ._lib import (DomainError, HepError, InvalidArgument, NcclError, RuntimeFailure,  # noqa: F401
                   CudaError, declared_symbols, lib)
from . import topology  # noqa: F401

__all__ = ["topology", "lib", "HepError", "DomainError", "InvalidArgument", "RuntimeFailure"]
