"""ctypes binding of the C-ABI in include/hep.h (libhep.so, built in-tree).

The product path has no fallback: if libhep.so is missing or fails to load, importing
this module raises.  Error codes are mapped back to the exception classes the
reference throws at the same points.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhep.so")

HEP_OK, HEP_ERR_DOMAIN, HEP_ERR_INVALID_ARGUMENT, HEP_ERR_RUNTIME = 0, 1, 2, 3
HEP_ERR_CUDA, HEP_ERR_NCCL, HEP_ERR_UNSUPPORTED = 4, 5, 6
HEP_F32, HEP_BF16 = 0, 1


class HepError(RuntimeError):
    """Base class; `code` is the hep_status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class DomainError(HepError, ValueError):
    """std::domain_error in the reference."""


class InvalidArgument(HepError, ValueError):
    """std::invalid_argument in the reference."""


class RuntimeFailure(HepError):
    """std::runtime_error in the reference (e.g. a corrupt SR wire)."""


class CudaError(HepError):
    pass


class NcclError(HepError):
    pass


_ERR = {
    HEP_ERR_DOMAIN: DomainError,
    HEP_ERR_INVALID_ARGUMENT: InvalidArgument,
    HEP_ERR_RUNTIME: RuntimeFailure,
    HEP_ERR_CUDA: CudaError,
    HEP_ERR_NCCL: NcclError,
}


class Level(C.Structure):
    _fields_ = [("scaling_factor", C.c_int64), ("domain_size", C.c_int64), ("bandwidth", C.c_double)]


class SrConfig(C.Structure):
    _fields_ = [
        ("ratio_CR", C.c_double),
        ("k", C.c_int64),
        ("index_width_bits", C.c_uint32),
        ("value_width_bits", C.c_uint32),
        ("per_matrix_budget", C.c_int),
    ]


class LayerParams(C.Structure):
    _fields_ = [
        ("hidden", C.c_int64),
        ("ffn", C.c_int64),
        ("experts", C.c_int64),
        ("top_k", C.c_int64),
        ("max_tokens", C.c_int64),
        ("dtype", C.c_int),
        ("levels", C.POINTER(Level)),
        ("num_levels", C.c_int),
        ("rank", C.c_int),
        ("use_sr", C.c_int),
        ("sr", SrConfig),
    ]


class Workload(C.Structure):
    _fields_ = [
        ("data_size_D", C.c_double),
        ("expert_size_PE", C.c_double),
        ("experts_per_gpu_n", C.c_int64),
        ("pre_blocks_m", C.c_int64),
        ("attn_latency", C.c_double),
        ("ffn_latency", C.c_double),
        ("expert_latency", C.c_double),
        ("backward_allreduce_const", C.c_double),
    ]


VP, I64, I32, SZ = C.c_void_p, C.c_int64, C.c_int, C.c_size_t
P = C.POINTER

# name -> argtypes (every function returns int hep_status unless listed in _RESTYPE)
SIGNATURES = {
    "hep_last_error": [],
    "hep_version": [],
    "hep_topology_gpus": [P(Level), I32, P(I64)],
    "hep_topology_build": [P(Level), I32, VP, VP],
    "hep_renumber": [P(Level), I32, I64, P(I64)],
    "hep_global_index": [P(Level), I32, P(I64), P(I64)],
    "hep_comm_type": [P(Level), I32, I64, I64, I32, P(I32)],
    "hep_level_frequency": [P(Level), I32, P(I64), P(I64)],
    "hep_traffic_report": [P(Level), I32, C.c_double, C.c_double, C.c_double,
                           P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double)],
    "hep_peer_lists": [P(Level), I32, I64, P(I64), P(I32), P(I32), P(I64), P(I32), P(I32)],
    "hep_route_table": [P(Level), I32, P(C.c_int32)],
    "hep_factor_domain_sizes": [I64, P(Level), I32, P(I64)],
    "hep_solve_optimal_p": [P(Workload), C.c_double, C.c_double, I64, P(C.c_double), P(I64), P(C.c_double)],
    "hep_plan_reports": [P(Level), I32, P(Workload), C.c_double, C.c_double, VP, C.c_char_p, P(C.c_double), P(I64),
                         P(C.c_double)],
    "hep_sr_resolve_k": [P(SrConfig), I64, I64, P(I64)],
    "hep_sr_wire_bytes": [I64, I64, P(SrConfig), P(SZ)],
    "hep_sr_workspace_bytes": [I64, I64, I32, P(SZ)],
    "hep_sr_encode": [VP, I32, VP, I64, I64, P(SrConfig), VP, SZ, VP, SZ, VP],
    "hep_sr_encode_batch": [P(VP), I32, I32, VP, I64, I64, P(SrConfig), P(VP), SZ, VP, SZ, VP],
    "hep_sr_encode_update_batch": [P(VP), P(VP), I32, C.c_float, VP, I64, I64, P(SrConfig), P(VP), SZ, VP, SZ, VP],
    "hep_sgd_step_batch": [P(VP), P(VP), I32, I64, C.c_float, VP],
    "hep_layer_sgd_step": [VP, P(VP), I32, C.c_float, VP],
    "hep_sr_decode": [VP, SZ, VP, I64, I64, VP, VP, VP],
    "hep_sr_decode_batch": [P(VP), I32, SZ, VP, I64, I64, P(VP), VP, VP],
    "hep_sr_check_status": [VP, VP],
    "hep_shared_mean": [P(VP), I32, I32, I64, VP, VP],
    "hep_comm_unique_id": [VP],
    "hep_comm_init": [VP, I32, I32, P(VP)],
    "hep_comm_init_virtual": [I32, P(VP)],
    "hep_comm_destroy": [VP],
    "hep_layer_create": [P(LayerParams), VP, P(VP)],
    "hep_layer_destroy": [VP],
    "hep_layer_set_gate": [VP, VP, I32, VP],
    "hep_layer_set_expert": [VP, I64, VP, VP, I32, VP],
    "hep_layer_set_shared": [VP, VP, VP],
    "hep_layer_refresh_shared": [VP, VP],
    "hep_layer_get_shared": [VP, VP, VP],
    "hep_layer_gather_experts": [VP, VP],
    "hep_layers_gather": [P(VP), I32, VP],
    "hep_layer_forward": [VP, VP, I64, VP, VP],
    "hep_layer_forward_residual": [VP, VP, I64, VP, VP],
    "hep_layer_forward_host": [VP, VP, I64, VP, VP],
    "hep_layer_host_fence": [VP, VP],
    "hep_layer_check": [VP, VP],
    "hep_layer_debug_corrupt_next_gather": [VP],
    "hep_layer_comm_bench": [VP, VP, I64, I32, P(C.c_double), VP],
    "hep_layer_debug": [VP, P(VP), P(VP), P(VP), P(VP), P(VP)],
    "hep_layer_set_profiling": [VP, I32],
    "hep_layer_timings": [VP, C.c_char_p, SZ, P(C.c_float), I32, P(I32)],
    "hep_layer_launch_count": [VP, P(I32)],
    "hep_layer_gemm_schedule": [VP, P(C.c_uint32), P(C.c_uint32)],
    "hep_route_plan": [P(Level), I32, I32, I32, VP, I64, I64, VP, I64, I64, VP, VP, VP, VP, VP],
    "hep_grouped_gemm": [I32, VP, I64, VP, I64, VP, I64, I64, VP, VP, VP, I32, I32, C.c_uint32, VP],
    "hep_transpose_convert": [I32, VP, I64, I64, I32, VP, VP],
}
_RESTYPE = {"hep_last_error": C.c_char_p, "hep_version": C.c_char_p}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the hot path)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPE.get(name, C.c_int)
    return lib


lib = _load()


def check(status: int) -> None:
    if status != HEP_OK:
        msg = lib.hep_last_error().decode(errors="replace")
        raise _ERR.get(status, HepError)(status, msg)


def declared_symbols(header: str | None = None) -> list[str]:
    """Every hep_* function declared in include/hep.h (used by the export test)."""
    import re

    header = header or os.path.join(os.path.dirname(_HERE), "include", "hep.h")
    text = open(header).read()
    return sorted(set(re.findall(r"\b(hep_[a-z0-9_]+)\s*\(", text)))
