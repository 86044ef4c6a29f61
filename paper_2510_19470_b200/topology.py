"""Python mirror of the reference planner API for the hot path (hybridep::topo /
hybridep plan / perf solver), calling the C++ implementation in libhep.so.

Names and argument meaning follow proj/include/hybridep/topology.hpp and plan.hpp;
errors raise the classes in _lib that mirror std::domain_error /
std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import Level, Workload, check, lib

NONE, AG, A2A = 0, 1, 2


@dataclass
class LevelSpec:
    scaling_factor: int = 1
    domain_size: int = 1
    bandwidth: float = 1e9


@dataclass
class ClusterSpec:
    levels: list = field(default_factory=list)  # outermost first

    @staticmethod
    def of(sf, sed=None, bandwidth=1e9) -> "ClusterSpec":
        sed = sed or [1] * len(sf)
        return ClusterSpec([LevelSpec(int(a), int(b), bandwidth) for a, b in zip(sf, sed)])

    def _c(self):
        arr = (Level * len(self.levels))(*[Level(l.scaling_factor, l.domain_size, l.bandwidth) for l in self.levels])
        return arr, len(self.levels)

    def total_gpus(self) -> int:
        arr, n = self._c()
        g = C.c_int64()
        check(lib.hep_topology_gpus(arr, n, C.byref(g)))
        return g.value

    def level_count(self) -> int:
        return len(self.levels)

    @property
    def sf(self):
        return [l.scaling_factor for l in self.levels]

    @property
    def sed(self):
        return [l.domain_size for l in self.levels]


def renumber(m: int, cluster: ClusterSpec) -> list[int]:
    arr, n = cluster._c()
    out = (C.c_int64 * n)()
    check(lib.hep_renumber(arr, n, m, out))
    return list(out)


def global_index(idx, cluster: ClusterSpec) -> int:
    arr, n = cluster._c()
    if len(idx) != n:
        # same failure class as the reference (domain_error on level-count mismatch)
        from ._lib import DomainError
        raise DomainError(1, "multi-index level count mismatch")
    x = (C.c_int64 * n)(*idx)
    m = C.c_int64()
    check(lib.hep_global_index(arr, n, x, C.byref(m)))
    return m.value


def comm_type(m: int, n: int, level: int, cluster: ClusterSpec) -> int:
    arr, L = cluster._c()
    t = C.c_int()
    check(lib.hep_comm_type(arr, L, m, n, level, C.byref(t)))
    return t.value


@dataclass
class Topology:
    """Dense topology table (CommTopology): level[m, n] (-1 none), type[m, n]."""
    cluster: ClusterSpec
    level: np.ndarray
    type: np.ndarray
    freq_a2a: list
    freq_ag: list

    def gpus(self) -> int:
        return self.level.shape[0]

    def classify(self, m: int, n: int):
        return int(self.level[m, n]), int(self.type[m, n])


def build_topology(cluster: ClusterSpec) -> Topology:
    arr, L = cluster._c()
    G = cluster.total_gpus()
    lvl = np.empty((G, G), np.int8)
    typ = np.empty((G, G), np.uint8)
    check(lib.hep_topology_build(arr, L, lvl.ctypes.data, typ.ctypes.data))
    a2a = (C.c_int64 * L)()
    ag = (C.c_int64 * L)()
    check(lib.hep_level_frequency(arr, L, a2a, ag))
    return Topology(cluster, lvl, typ, list(a2a), list(ag))


def traffic_report(cluster: ClusterSpec, data_size_D: float, expert_size_PE: float, token_multiplier=1.0):
    arr, L = cluster._c()
    outs = [(C.c_double * L)() for _ in range(4)]
    check(lib.hep_traffic_report(arr, L, data_size_D, expert_size_PE, token_multiplier, *outs))
    return {"a2a_pair_bytes": list(outs[0]), "ag_pair_bytes": list(outs[1]),
            "a2a_bytes": list(outs[2]), "ag_bytes": list(outs[3])}


def peer_lists(cluster: ClusterSpec, m: int):
    """(ag, a2a): lists of (peer, level) in ring order (simcore.cpp:30-74)."""
    arr, L = cluster._c()
    G = cluster.total_gpus()
    ag, agl, a2a, a2al = (C.c_int64 * G)(), (C.c_int * G)(), (C.c_int64 * G)(), (C.c_int * G)()
    na, nb = C.c_int(), C.c_int()
    check(lib.hep_peer_lists(arr, L, m, ag, agl, C.byref(na), a2a, a2al, C.byref(nb)))
    return [(ag[i], agl[i]) for i in range(na.value)], [(a2a[i], a2al[i]) for i in range(nb.value)]


def route_table(cluster: ClusterSpec) -> np.ndarray:
    arr, L = cluster._c()
    G = cluster.total_gpus()
    out = np.empty((G, G), np.int32)
    check(lib.hep_route_table(arr, L, out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def factor_domain_sizes(domain_size: int, cluster: ClusterSpec) -> list[int]:
    arr, L = cluster._c()
    out = (C.c_int64 * L)()
    check(lib.hep_factor_domain_sizes(domain_size, arr, L, out))
    return list(out)


def solve_optimal_p(*, data_size_D, expert_size_PE, experts_per_gpu_n, pre_blocks_m, attn_latency,
                    ffn_latency, expert_latency, backward_allreduce_const=0.0, throughput_C, bandwidth_B, gpus):
    w = Workload(data_size_D, expert_size_PE, experts_per_gpu_n, pre_blocks_m, attn_latency, ffn_latency,
                 expert_latency, backward_allreduce_const)
    p, s, lat = C.c_double(), C.c_int64(), (C.c_double * 6)()
    check(lib.hep_solve_optimal_p(C.byref(w), throughput_C, bandwidth_B, gpus, C.byref(p), C.byref(s), lat))
    keys = ("comp", "pre_expert", "comm_a2a", "comm_ag", "overlap", "total")
    return p.value, s.value, dict(zip(keys, list(lat)))


def plan_reports(cluster: ClusterSpec, *, data_size_D, expert_size_PE, experts_per_gpu_n, attn_latency,
                 expert_latency, throughput_C, bandwidth_B, pre_blocks_m=0, ffn_latency=1e-12, pinned_sed=None,
                 out_dir=None):
    """The reference's plan + topo reports (plan.json, freq.json, topo.csv) for measured
    inputs (hep_plan_reports): returns (p, per-level S_ED, latency terms)."""
    w = Workload(data_size_D, expert_size_PE, experts_per_gpu_n, pre_blocks_m, attn_latency, ffn_latency,
                 expert_latency, 0.0)
    arr, n = cluster._c()
    pin = (C.c_int64 * n)(*pinned_sed) if pinned_sed is not None else None
    p = C.c_double()
    sed = (C.c_int64 * n)()
    lat = (C.c_double * 6)()
    check(lib.hep_plan_reports(arr, n, C.byref(w), throughput_C, bandwidth_B, pin, (out_dir or "").encode(),
                               C.byref(p), sed, lat))
    keys = ("comp", "pre_expert", "comm_a2a", "comm_ag", "overlap", "total")
    return p.value, list(sed), dict(zip(keys, list(lat)))
