"""ORACLE — test infrastructure only (see moe_oracle.c header).

Python access to
  * `orc`: the CPU restatement (oracle/_build/liboracle.so), and
  * `ref`: the unmodified reference library (oracle/_ref/libhybridep_ref.so), when built.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libhybridep_ref.so")


def build() -> None:
    subprocess.run(["make", "-C", HERE, "-s"], check=True)


def _load_orc():
    if not os.path.exists(ORC_PATH):
        build()
    lib = C.CDLL(ORC_PATH)
    I64, VP = C.c_int64, C.c_void_p
    lib.orc_gpus.restype = I64
    lib.orc_gpus.argtypes = [VP, C.c_int]
    lib.orc_renumber.argtypes = [VP, C.c_int, I64, VP]
    lib.orc_renumber.restype = None
    lib.orc_topology.argtypes = [VP, VP, C.c_int, VP, VP]
    lib.orc_topology.restype = None
    lib.orc_peer_lists.argtypes = [VP, VP, C.c_int, I64, VP, VP, VP, VP, VP, VP]
    lib.orc_peer_lists.restype = None
    lib.orc_route_table.argtypes = [VP, VP, C.c_int, VP]
    lib.orc_shared_mean.argtypes = [VP, C.c_int, I64, VP]
    lib.orc_shared_mean.restype = None
    lib.orc_resolve_k.restype = I64
    lib.orc_resolve_k.argtypes = [C.c_double, I64, C.c_uint32, C.c_uint32, I64, I64]
    lib.orc_sr_encode.restype = I64
    lib.orc_sr_encode.argtypes = [VP, VP, I64, I64, C.c_double, I64, C.c_uint32, C.c_uint32, C.c_int, VP]
    lib.orc_sr_decode.argtypes = [VP, I64, VP, I64, I64, VP]
    lib.orc_gate.argtypes = [VP, VP, I64, I64, I64, I64, VP, VP]
    lib.orc_gate.restype = None
    lib.orc_moe_layer.argtypes = [C.c_int, VP, VP, VP, VP, I64, I64, I64, I64, I64, I64, VP, VP, C.c_int, I64,
                                  VP, VP, VP, VP, VP]
    lib.orc_num_threads.restype = C.c_int
    lib.orc_ffn_row.argtypes = [VP, VP, VP, I64, I64, C.c_int, VP, VP, VP]
    lib.orc_ffn_row.restype = None
    lib.orc_sgd_step.argtypes = [VP, VP, C.c_float, I64]
    lib.orc_sgd_step.restype = None
    return lib


orc = _load_orc()


def _load_ref():
    if not os.path.exists(REF_PATH):
        return None
    lib = C.CDLL(REF_PATH)
    I64, VP, D = C.c_int64, C.c_void_p, C.c_double
    lib.ref_topology.argtypes = [VP, VP, C.c_int, VP, VP]
    lib.ref_renumber.argtypes = [VP, C.c_int, I64, VP]
    lib.ref_global_index.argtypes = [VP, C.c_int, VP, C.c_int, VP]
    lib.ref_comm_type.argtypes = [VP, VP, C.c_int, I64, I64, C.c_int, VP]
    lib.ref_level_frequency.argtypes = [VP, VP, C.c_int, VP, VP]
    lib.ref_traffic_report.argtypes = [VP, VP, C.c_int, D, D, D, VP]
    lib.ref_factor_domain_sizes.argtypes = [I64, VP, C.c_int, VP]
    lib.ref_schedule.restype = I64
    lib.ref_schedule.argtypes = [VP, VP, C.c_int, D, D, I64, D, D, D, D, C.c_int, I64, VP, VP, VP, I64, VP]
    lib.ref_solve_optimal_p.argtypes = [D, D, I64, I64, D, D, D, D, D, D, I64, VP, VP, VP]
    lib.ref_sr_resolve_k.restype = I64
    lib.ref_sr_resolve_k.argtypes = [D, I64, C.c_uint32, C.c_uint32, I64, I64]
    lib.ref_sr_encode.restype = I64
    lib.ref_sr_encode.argtypes = [VP, VP, I64, I64, D, I64, C.c_uint32, C.c_uint32, C.c_int, VP, I64]
    lib.ref_sr_decode.argtypes = [VP, I64, VP, I64, I64, VP]
    lib.ref_shared_mean.argtypes = [VP, C.c_int, I64, I64, VP]
    lib.ref_sim_step.argtypes = [VP, VP, C.c_int, D, D, D, I64, D, D, D, D, C.c_int, VP, VP]
    return lib


ref = _load_ref()


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------- topology
def topology(sf, sed, lib=None):
    lib = lib or orc
    sf_, sed_ = _i64(sf), _i64(sed)
    G = int(np.prod(sf_))
    lvl = np.empty((G, G), np.int8)
    typ = np.empty((G, G), np.uint8)
    fn = lib.orc_topology if lib is orc else lib.ref_topology
    fn(_p(sf_), _p(sed_), len(sf_), _p(lvl), _p(typ))
    return lvl, typ


def peer_lists(sf, sed, m):
    sf_, sed_ = _i64(sf), _i64(sed)
    G = int(np.prod(sf_))
    ag, a2a = np.zeros(G, np.int64), np.zeros(G, np.int64)
    agl, a2al = np.zeros(G, np.int32), np.zeros(G, np.int32)
    na, nb = C.c_int(), C.c_int()
    orc.orc_peer_lists(_p(sf_), _p(sed_), len(sf_), m, _p(ag), _p(agl), C.byref(na), _p(a2a), _p(a2al), C.byref(nb))
    return list(zip(ag[: na.value].tolist(), agl[: na.value].tolist())), \
        list(zip(a2a[: nb.value].tolist(), a2al[: nb.value].tolist()))


def route_table(sf, sed):
    sf_, sed_ = _i64(sf), _i64(sed)
    G = int(np.prod(sf_))
    out = np.empty((G, G), np.int32)
    rc = orc.orc_route_table(_p(sf_), _p(sed_), len(sf_), _p(out))
    if rc:
        raise ValueError("route table has a hole")
    return out


def sim_step(sf, sed, bandwidth, D, PE, n, pre, expert_lat, enc=0.0, dec=0.0, layers=1):
    """The reference's own step DAG + discrete-event engine (oracle/_ref): (makespan s,
    worst All-Gather stall s)."""
    if ref is None:
        raise RuntimeError("oracle/_ref/libhybridep_ref.so is not built (needs /root/reference once)")
    sf_, sed_ = _i64(sf), _i64(sed)
    mk, st = C.c_double(), C.c_double()
    rc = ref.ref_sim_step(_p(sf_), _p(sed_), len(sf_), float(bandwidth), float(D), float(PE), int(n), float(pre),
                          float(expert_lat), float(enc), float(dec), int(layers), C.byref(mk), C.byref(st))
    if rc:
        raise ValueError(f"reference sim failed ({rc})")
    return mk.value, st.value


# --------------------------------------------------------------------- SR codec
def wire_size(P, k, iw=32, vw=32):
    return 28 + k * (iw + vw) // 8


def sr_encode(expert, shared, h, m, ratio=None, k=None, iw=32, vw=32, per_matrix=False, use_ref=False):
    expert = np.ascontiguousarray(expert, np.float32)
    shared = np.ascontiguousarray(shared, np.float32)
    P = 2 * h * m
    kk = orc.orc_resolve_k(float(ratio or 1.0), -1 if k is None else int(k), iw, vw, P, 4)
    cap = wire_size(P, kk, iw, vw)
    wire = np.zeros(cap, np.uint8)
    if use_ref:
        n = ref.ref_sr_encode(_p(expert), _p(shared), h, m, float(ratio or 1.0), -1 if k is None else int(k), iw, vw,
                              int(per_matrix), _p(wire), cap)
    else:
        n = orc.orc_sr_encode(_p(expert), _p(shared), h, m, float(ratio or 1.0), -1 if k is None else int(k), iw, vw,
                              int(per_matrix), _p(wire))
    if n < 0:
        raise ValueError(f"encode failed ({n})")
    return wire[:n]


def sr_decode(wire, shared, h, m, use_ref=False):
    wire = np.ascontiguousarray(wire, np.uint8)
    shared = np.ascontiguousarray(shared, np.float32)
    out = np.zeros(2 * h * m, np.float32)
    fn = ref.ref_sr_decode if use_ref else orc.orc_sr_decode
    rc = fn(_p(wire), wire.size, _p(shared), h, m, _p(out))
    return rc, out


def sgd_step(master, grad, lr):
    """m - lr g with one rounding (fmaf), as the fused encode applies it."""
    m = np.ascontiguousarray(master, np.float32).copy()
    g = np.ascontiguousarray(grad, np.float32)
    orc.orc_sgd_step(_p(m), _p(g), float(lr), m.size)
    return m


def shared_mean(experts, use_ref=False, h=None, m=None):
    arrs = [np.ascontiguousarray(e, np.float32) for e in experts]
    P = arrs[0].size
    out = np.zeros(P, np.float32)
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    if use_ref:
        ref.ref_shared_mean(ptrs, len(arrs), h, m, _p(out))
    else:
        orc.orc_shared_mean(ptrs, len(arrs), P, _p(out))
    return out


# --------------------------------------------------------------------- MoE layer
def gate(x, wg, k):
    x = np.ascontiguousarray(x, np.float32)
    wg = np.ascontiguousarray(wg, np.float32)
    T, H = x.shape
    E = wg.shape[1]
    idx = np.zeros((T, k), np.int32)
    w = np.zeros((T, k), np.float32)
    orc.orc_gate(_p(x), _p(wg), T, H, E, k, _p(idx), _p(w))
    return idx, w


def moe_layer(x, wg, w_up, w_down, k, sf, sed, bf16, stride=1, exact=False):
    """x: [G, T, H]; wg: [H, E]; w_up: [E, H, F]; w_down: [E, F, H] (fp32 values).
    bf16=True mirrors the device's bf16 rounding points; with exact=True a bf16 layer is
    instead evaluated as the fp32 reference (same bf16 routing, h and y unrounded).
    Returns dict(y [G,T,H], topk_idx, topk_w, pos [G,T,k], key_counts [G, G*E])."""
    x = np.ascontiguousarray(x, np.float32)
    wg = np.ascontiguousarray(wg, np.float32)
    w_up = np.ascontiguousarray(w_up, np.float32)
    w_down = np.ascontiguousarray(w_down, np.float32)
    G, T, H = x.shape
    E, _, F = w_up.shape
    sf_, sed_ = _i64(sf), _i64(sed)
    y = np.zeros((G, T, H), np.float32)
    ti = np.zeros((G, T, k), np.int32)
    tw = np.zeros((G, T, k), np.float32)
    pos = np.zeros((G, T, k), np.int32)
    kc = np.zeros((G, G * E), np.int32)
    mode = (2 if exact else 1) if bf16 else 0
    rc = orc.orc_moe_layer(mode, _p(x), _p(wg), _p(w_up), _p(w_down), G, T, H, F, E, k, _p(sf_), _p(sed_),
                           len(sf_), stride, _p(y), _p(ti), _p(tw), _p(pos), _p(kc))
    if rc:
        raise ValueError(f"oracle layer failed ({rc})")
    return {"y": y, "topk_idx": ti, "topk_w": tw, "pos": pos, "key_counts": kc}


def ffn_row(x, w_up, w_down, bf16):
    """S4 for one row (the per-row definition): y = relu(x w_up) w_down, fp64 sums."""
    x = np.ascontiguousarray(x, np.float32)
    w_up = np.ascontiguousarray(w_up, np.float32)
    w_down = np.ascontiguousarray(w_down, np.float32)
    H, F = w_up.shape
    hacc, yacc = np.zeros(F), np.zeros(H)
    out = np.zeros(H, np.float32)
    orc.orc_ffn_row(_p(x), _p(w_up), _p(w_down), H, F, int(bf16), _p(hacc), _p(yacc), _p(out))
    return out


def num_threads() -> int:
    return orc.orc_num_threads()
