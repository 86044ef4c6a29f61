"""Table of the config sweep (tools/sweep_configs.sh): tokens/s, e2e, GEMM roofline, bus GB/s."""
import glob
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep"
rows = []
for f in sorted(glob.glob(os.path.join(d, "*.log"))):
    line = None
    for ln in open(f):
        if ln.startswith("{") and '"metric"' in ln:
            line = json.loads(ln)
    name = os.path.basename(f)[:-4]
    if line is None:
        rows.append(f"| {name} | (no JSON line) |")
        continue
    c = line["config"]
    comm = line.get("comm") or {}
    roof = line.get("roofline") or {}
    rows.append("| {} | {} | {} | {} | {:.3f} M | {:.3f} M | {:.1f} ms | {} | {} | {} |".format(
        name, line["n_gpus"], c.get("sf"), c.get("sed"), line["value"] / 1e6, line["e2e"]["value"] / 1e6,
        line["ms_per_step"], f"{roof.get('achieved', 0):.0f} ({roof.get('frac', 0):.2f})" if roof else "-",
        f"{comm.get('a2a_bus_gbs', 0):.0f} / {comm.get('ag_bus_gbs', 0):.0f}" if comm else "-",
        line.get("clocks", {}).get("sm_mhz")))
print("| run | N | SF | S_ED | tokens/s | e2e tokens/s | ms/step | GEMM TF/s (frac) | A2A / AG bus GB/s | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
