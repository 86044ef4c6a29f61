"""Generates tests/golden/ fixtures from the UNMODIFIED reference (oracle/_ref), so the
GPU boxes (which have no /root/reference) test against the reference's own outputs.

    python oracle/gen_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from tests.test_host import hierarchies  # noqa: E402


def ref_peer_lists(sf, sed):
    """Peer order as the reference emits it: the AgTransfer / A2aDispatch jobs of
    build_schedule (simcore.cpp:155-202) list each GPU's peers in ring order."""
    import ctypes as C
    sf_, sed_ = oracle._i64(sf), oracle._i64(sed)
    cap = 4096
    rows = np.zeros((cap, 6), np.int64)
    bd = np.zeros((cap, 2), np.float64)
    deps = np.zeros(cap * 16, np.int64)
    nd = C.c_int64()
    n = oracle.ref.ref_schedule(oracle._p(sf_), oracle._p(sed_), len(sf), 8e6, 2e6, 1, 1e-3, 1e-3, 0.0, 0.0, 1, cap,
                                oracle._p(rows), oracle._p(bd), oracle._p(deps), deps.size, C.byref(nd))
    G = int(np.prod(sf))
    ag = [[] for _ in range(G)]
    a2a = [[] for _ in range(G)]
    for r in rows[:n]:
        kind, _, _, gpu, peer, _ = r.tolist()
        if kind == 3:
            ag[gpu].append(peer)
        elif kind == 4:
            a2a[gpu].append(peer)
    return ag, a2a


def main():
    assert oracle.ref is not None, "build oracle/_ref first (make -C oracle)"
    out = []
    import ctypes as C
    for sf, sed in hierarchies(8):
        lvl, typ = oracle.topology(sf, sed, lib=oracle.ref)
        L = len(sf)
        a2a_f, ag_f = np.zeros(L, np.int64), np.zeros(L, np.int64)
        oracle.ref.ref_level_frequency(oracle._p(oracle._i64(sf)), oracle._p(oracle._i64(sed)), L,
                                       oracle._p(a2a_f), oracle._p(ag_f))
        tr = np.zeros(4 * L)
        oracle.ref.ref_traffic_report(oracle._p(oracle._i64(sf)), oracle._p(oracle._i64(sed)), L, 4194304.0,
                                      33554432.0, 1.0, oracle._p(tr))
        ag, a2a = ref_peer_lists(sf, sed)
        out.append({"sf": sf, "sed": sed, "level": lvl.tolist(), "type": typ.tolist(),
                    "freq_a2a": a2a_f.tolist(), "freq_ag": ag_f.tolist(),
                    "ag_peers": ag, "a2a_peers": a2a,
                    "a2a_bytes": tr[2::4].tolist(), "ag_bytes": tr[3::4].tolist()})
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    with open(os.path.join(ROOT, "tests", "golden", "topology_g8.json"), "w") as f:
        json.dump(out, f)

    # SR codec fixtures: seeded demo experts -> reference wire bytes and decoded experts.
    rng = np.random.default_rng(2024)
    cases = {}
    specs = [(4, 6, None, 10, 32, 32, 0), (8, 12, 50.0, None, 32, 32, 0), (8, 12, None, 37, 64, 64, 1),
             (16, 16, 10.0, None, 32, 64, 1), (3, 5, None, 0, 32, 32, 0), (3, 5, None, 1000, 64, 32, 0)]
    for i, (h, m, ratio, k, iw, vw, pm) in enumerate(specs):
        P = 2 * h * m
        base = (0.05 + 0.95 * rng.random(P)) * np.where(rng.random(P) < 0.5, -1, 1)
        e = (base + rng.uniform(-0.05, 0.05, P)).astype(np.float32)
        s = base.astype(np.float32)
        if i % 2:
            e = (s + np.round(rng.uniform(-3, 3, P)) / 32).astype(np.float32)  # ties
        wire = oracle.sr_encode(e, s, h, m, ratio=ratio, k=k, iw=iw, vw=vw, per_matrix=bool(pm), use_ref=True)
        rc, dec = oracle.sr_decode(wire, s, h, m, use_ref=True)
        assert rc == 0
        cases[f"c{i}_expert"] = e
        cases[f"c{i}_shared"] = s
        cases[f"c{i}_wire"] = wire
        cases[f"c{i}_decoded"] = dec
        cases[f"c{i}_spec"] = np.array([h, m, -1 if ratio is None else ratio, -1 if k is None else k, iw, vw, pm],
                                       np.float64)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "sr_cases.npz"), **cases)

    # Planner reports: the reference's own run_plan + run_topo (oracle/_ref/ref_reports)
    # on B200-like measured inputs (D, P_E, n, pre-expert s, expert s, C FLOP/s, B bytes/s).
    import subprocess
    import tempfile
    reports = []
    for sf, pin, D, PE, n, pre, ex, Cc, B in [
            ([2], None, 2.68e8, 9.4e8, 4, 1.7e-4, 6.9e-4, 1.4e15, 7.4e11),
            ([2, 2], None, 2.68e8, 4.7e8, 2, 1.7e-4, 1.4e-3, 1.4e15, 7.4e11),
            ([2, 4], None, 2.68e8, 2.35e8, 1, 1.7e-4, 2.7e-3, 1.4e15, 7.4e11),
            ([2, 4], [1, 4], 2.68e8, 2.35e8, 1, 1.7e-4, 2.7e-3, 1.4e15, 7.4e11),
            ([2, 4], None, 4.0e6, 2.35e8, 1, 2.0e-3, 2.0e-5, 1.4e15, 7.4e11),   # tiny token volume: AG wins
            ([2, 2, 2], None, 2.0e8, 1.8e6, 8, 1.0e-4, 5.0e-5, 1.4e15, 7.4e11),
            ([2, 2, 2], [1, 2, 2], 2.0e8, 1.8e6, 8, 1.0e-4, 5.0e-5, 1.4e15, 7.4e11)]:
        with tempfile.TemporaryDirectory() as d:
            args = [os.path.join(HERE, "_ref", "ref_reports"), d] + [repr(v) for v in (D, PE, n, pre, ex, Cc, B)] + \
                   [",".join(map(str, sf))] + ([",".join(map(str, pin))] if pin else [])
            subprocess.run(args, check=True, capture_output=True)
            reports.append({"sf": sf, "pinned_sed": pin, "D": D, "PE": PE, "n": n, "pre": pre, "expert": ex, "C": Cc,
                            "B": B, "plan": json.load(open(os.path.join(d, "plan.json"))),
                            "freq": json.load(open(os.path.join(d, "freq.json"))),
                            "topo_csv": open(os.path.join(d, "topo.csv")).read()})
    with open(os.path.join(ROOT, "tests", "golden", "plan_reports.json"), "w") as f:
        json.dump(reports, f, indent=1)
    print("wrote tests/golden/topology_g8.json, sr_cases.npz and plan_reports.json")


if __name__ == "__main__":
    main()
