"""The reference's latency model for every S_ED of a measured cfg5 sweep, with and without
a load-imbalance term, against the measured step (profiles/r2_cfg5_sweep/).

The reference's model (perfmodel.cpp:141-153, via hep_plan_reports with the hierarchy
pinned) assumes evenly activated experts: its compute term does not depend on S_ED.  The
extension adds comp * (imbalance - 1), imbalance = the measured busiest-GPU rows / mean
rows of each layer, averaged over the stack.  CPU only (host planner in libhep).

    python tools/model_imbalance.py [--sweep profiles/r2_cfg5_sweep] [--planner-log profiles/r2_final2/cfg5_n4.log]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_19470_b200 import topology as topo  # noqa: E402


def line(path):
    for l in open(path):
        if l.startswith("{"):
            return json.loads(l)
    raise ValueError(path)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", default=os.path.join(ROOT, "profiles", "r2_cfg5_sweep"))
    ap.add_argument("--planner-log", default=os.path.join(ROOT, "profiles", "r2_final2", "cfg5_n4.log"))
    a = ap.parse_args()
    inp = line(a.planner_log)["planner"]["measured_inputs"]
    H, F, E, k, T, b, L = 4096, 14336, 8, 2, 16384, 2, 8
    sf, world = [2, 2], 4
    n = E // world
    rows = T * k
    rows_out = []
    for sed in ([1, 1], [2, 1], [1, 2], [2, 2]):
        d = line(os.path.join(a.sweep, "cfg5_n4_sed%d%d.log" % tuple(sed)))
        p, got, lat = topo.plan_reports(
            topo.ClusterSpec.of(sf, [1] * len(sf), bandwidth=inp["nvlink_bytes_per_s"]),
            data_size_D=float(rows * H * b), expert_size_PE=float(n * 2 * H * F * b), experts_per_gpu_n=n,
            attn_latency=inp["pre_expert_s"], expert_latency=inp["expert_s_per_routed_row"] * rows / n,
            throughput_C=inp["gemm_flops_per_s"], bandwidth_B=inp["nvlink_bytes_per_s"], pinned_sed=sed)
        imb = sum(d["layer_load_imbalance"]) / len(d["layer_load_imbalance"])
        adj = lat["total"] + lat["comp"] * (imb - 1.0)
        rows_out.append({"sed": sed, "p": p, "model_ms_per_layer": lat["total"] * 1e3, "imbalance": imb,
                         "model_with_imbalance_ms_per_layer": adj * 1e3,
                         "measured_ms_per_layer": d["ms_per_step"] / L, "tokens_per_s": d["value"]})
    for r in rows_out:
        print(json.dumps(r))
    by = lambda key: [r["sed"] for r in sorted(rows_out, key=lambda r: r[key])]
    print(json.dumps({"rank_model": by("model_ms_per_layer"), "rank_model_with_imbalance": by("model_with_imbalance_ms_per_layer"),
                      "rank_measured": by("measured_ms_per_layer")}))


if __name__ == "__main__":
    main()
