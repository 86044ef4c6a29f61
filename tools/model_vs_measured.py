"""The paper's performance model next to the measured B200 step.

For every N>1 bench line in a directory (default profiles/r1_sweep), the reference's
step DAG (build_schedule, simcore.cpp:96-266) is built for the measured configuration
and run on the reference's own discrete-event engine (sim::run, from oracle/_ref: the
timing model is the reference's, not shipped by the B200 build) with MEASURED inputs:
  * pre-expert time      = gate + scans of that line + the N=1 permute of the config;
  * expert_latency       = that line's expert-GEMM time per layer / n;
  * NVLink bandwidth     = that line's measured A2A bus GB/s (AG bus GB/s if no A2A);
  * D = T*k*H*b, P_E = n * expert bytes (SR wire bytes for SR-migrated configs);
  * SR encode/decode per expert from profiles/r1_bench_sr_v2.log.
The predicted makespan (+ the measured combine, which the DAG does not model) is
compared with the measured ms/step.  Where they differ, the table says where the B200
implementation departs from the model's assumptions (e.g. the fp32 path's All-Gather
runs in-line over NCCL, while the model prefetches it from t=0).

    python tools/model_vs_measured.py [dir ...] > profiles/r1_model_vs_measured.md
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (the reference's engine, compiled from its sources)


def lines(dirs):
    out = []
    for d in dirs:
        for f in sorted(glob.glob(os.path.join(d, "*.log"))):
            for ln in open(f):
                if ln.startswith("{") and '"metric"' in ln and '"impl"' not in ln:
                    rec = json.loads(ln)
                    rec["_file"] = os.path.relpath(f, ROOT)
                    out.append(rec)
    return out


def sr_costs():
    p = os.path.join(ROOT, "profiles", "r1_bench_sr_v2.log")
    costs = {}
    if os.path.exists(p):
        for ln in open(p):
            if ln.startswith("{"):
                d = json.loads(ln)
                costs[d["shape"]] = (d["encode_batch_ms"] / d["batch"] / 1e3, d["decode_batch_ms"] / d["batch"] / 1e3)
    return costs


def main():
    dirs = sys.argv[1:] or [os.path.join(ROOT, "profiles", "r1_sweep")]
    recs = lines(dirs)
    n1 = {r["config"]["workload"].split(":")[0]: r for r in recs if r["n_gpus"] == 1}
    sr = sr_costs()
    print("| run | N | SF | S_ED | measured ms/step | model ms (DAG + combine) | error | AG stall (model) |")
    print("|---|---|---|---|---|---|---|---|")
    for r in recs:
        if r["n_gpus"] < 2:
            continue
        c = r["config"]
        name = c["workload"].split(":")[0]
        H, F, E, k, T = c["hidden"], c["ffn"], c["experts"], c["top_k"], c["tokens_per_gpu"]
        G = r["n_gpus"]
        layers = c.get("layers", 1)
        b = 2 if r["dtype"] == "bf16" else 4
        n = E // G
        ph = r["phase_ms"]
        gemm = sum(v for kk, v in ph.items() if kk.startswith("gemm_")) / layers / 1e3
        permute = n1[name]["phase_ms"].get("permute", 0.0) / 1e3 if name in n1 else 0.0
        pre = (ph.get("gate", 0.0) + ph.get("scan", 0.0)) / layers / 1e3 + permute
        comm = r.get("comm") or {}
        # the line's measured A2A bus GB/s; with no A2A, the AG bus GB/s of dense experts,
        # and for SR wires the copy-engine pull rate (the line's AG figure folds the
        # encode/decode time in; the DAG models those separately)
        bw = comm.get("a2a_bus_gbs") or (724.0 if c.get("sr_migration") else comm.get("ag_bus_gbs")) or 700.0
        bw *= 1e9
        P = 2 * H * F
        if c.get("sr_migration"):
            k_sr = P * 4 // (50 * 8)
            pe = n * (28 + 8 * k_sr)
            enc, dec = sr.get(name, (0.0, 0.0))
        else:
            pe = n * P * b
            enc = dec = 0.0
        mk, stall = oracle.sim_step(c["sf"], c["sed"], bw, D=T * k * H * b, PE=pe, n=n, pre=pre,
                                    expert_lat=gemm / n, enc=enc, dec=dec, layers=layers)
        combine = ph.get("combine", 0.0) / 1e3  # all layers
        model = (mk + combine) * 1e3
        meas = r["ms_per_step"]
        print(f"| {os.path.basename(r['_file'])[:-4]} | {G} | {c['sf']} | {c['sed']} | {meas:.3f} | {model:.3f} | "
              f"{(model - meas) / meas:+.1%} | {stall * 1e3:.3f} |")


if __name__ == "__main__":
    main()
