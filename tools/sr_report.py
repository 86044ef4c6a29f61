"""Summarise tools/gpu_sr_check.sh output: bench_sr lines and the SR kernels' launch list."""
import csv
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "v"
for line in open(f"gpurun_out/bench_sr_{tag}.log"):
    if line.startswith("{"):
        d = json.loads(line)
        print(d["shape"], "encode %.3f ms (%.2f of HBM)  batch8 %.3f ms (%.2f)  decode %.3f ms (%.2f)" % (
            d["encode_ms"], d["encode_frac"], d["encode_batch_ms"], d["encode_batch_frac"], d["decode_ms"],
            d["decode_frac"]))
rows = list(csv.DictReader(line for line in open(f"gpurun_out/sr_launches_{tag}.csv") if line.startswith('"')))
for r in rows:
    if r["Metric Name"] == "gpu__time_duration.sum" and "sr_" in r["Kernel Name"]:
        print(r["ID"], r["Kernel Name"].split("(")[0].split("::")[-1], r["Grid Size"], r["Metric Value"])
