"""Per-kernel roofline table of one MoE-layer forward (N=1), from an ncu launch list.

    # on the GPU box (the ncu pass is separate from any timed run):
    python tools/kernel_roofline.py run --config cfg3            # exits 0 without ncu first
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --clock-control none --csv --log-file gpurun_out/kr_cfg3.csv \\
        python tools/kernel_roofline.py run --config cfg3
    # anywhere:
    python tools/kernel_roofline.py report --config cfg3 --csv gpurun_out/kr_cfg3.csv

The forward runs twice; the report takes the second one.  Achieved = the kernel's
ALGORITHMIC bytes / its ncu duration, against the HBM copy peak of
MEASURED_PEAKS.json; the GEMMs are reported in TFLOP/s against the bf16 peaks.  ncu's
per-launch times are serialised and cold-cache, so these are per-kernel ceilings, not
the in-step share (bench.py's phase_ms is).  DRAM bytes show re-reads beyond the
algorithmic traffic.
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def run(cfg_name):
    import torch

    from paper_2510_19470_b200.moe import MoELayer

    cfg = bench.CONFIGS[cfg_name]
    dev = torch.device("cuda", 0)
    dtype = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    x, wg = bench.make_inputs(cfg, 0, dev, dtype)
    layer = MoELayer(hidden=cfg["H"], ffn=cfg["F"], experts=cfg["E"], top_k=cfg["k"], max_tokens=cfg["T"],
                     dtype=dtype, sf=[1], sed=[1], rank=0)
    layer.set_gate(wg)
    for e in layer.owned_experts():
        u, d = bench.expert_weights(cfg, e, dev, dtype)
        layer.set_expert(e, u, d)
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    for _ in range(2):
        layer.forward(x, out=y)
    torch.cuda.synchronize()
    print("ok", flush=True)


def kind(name):
    n = name.split("(")[0]
    for key, k in (("gate", "K1 gate"), ("chunk_scan", "scan"), ("key_scan", "scan"), ("positions", "scan"),
                   ("permute", "K2 permute"), ("grouped_gemm", "K8 grouped GEMM"), ("gemm_f32", "K8 grouped GEMM"),
                   ("combine", "K9 combine")):
        if key in n:
            return k
    return None


def report(cfg_name, path):
    cfg = bench.CONFIGS[cfg_name]
    peaks = bench.peaks()  # MEASURED_PEAKS.json (driver-written), else the recipe's fallback
    hbm = peaks["hbm_gbs"]
    T, H, F, E, k = cfg["T"], cfg["H"], cfg["F"], cfg["E"], cfg["k"]
    b = 2 if cfg["dtype"] == "bf16" else 4
    launches = {}
    order = []
    for r in csv.DictReader(line for line in open(path) if line.startswith('"')):
        key = r["ID"]
        if key not in launches:
            launches[key] = {"name": r["Kernel Name"]}
            order.append(key)
        scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r.get("Metric Unit", ""), 1.0)
        launches[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale  # ns / bytes
    ours = [launches[i] for i in order if kind(launches[i]["name"])]
    gates = [i for i, l in enumerate(ours) if kind(l["name"]) == "K1 gate"]
    fwd = ours[gates[-1]:] if gates else ours
    rows = T * k
    alg = {  # algorithmic bytes per launch
        "K1 gate": T * H * b + H * E * 4 + T * k * 8,
        "K2 permute": T * H * b + rows * H * b + rows * 4,
        "K9 combine": rows * H * b + rows * 4 + rows * 4 + T * H * b,
    }
    out = []
    gemm_i = 0
    for l in fwd:
        kd = kind(l["name"])
        ms = l.get("gpu__time_duration.sum", 0.0) / 1e6
        dram = l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
        rec = {"kernel": l["name"].split("(")[0].split("::")[-1], "kind": kd, "ms": ms, "dram_bytes": dram}
        if kd == "K8 grouped GEMM":
            flops = 2.0 * rows * H * F
            # fp32 layers run 3xTF32: tf32 is half the bf16 rate and takes three passes, so
            # the fp32 peak is bf16/6; the hi/lo operand pairs it streams are 2x the fp32 bytes
            peak = peaks["bf16_tflops"] / (1 if b == 2 else 6)
            rec.update(which="up" if gemm_i == 0 else "down", tflops=flops / ms / 1e9,
                       frac_burst=flops / ms / 1e9 / peak,
                       alg_bytes=(rows * H * b + E * H * F * b + rows * F * b) if gemm_i == 0 else
                       (rows * F * b + E * H * F * b + rows * H * b))
            if b == 4:
                rec.update(operand_bytes=2 * rec["alg_bytes"], operand_frac=2 * rec["alg_bytes"] / ms / 1e6 / hbm)
            gemm_i += 1
        elif kd in alg:
            rec.update(alg_bytes=alg[kd], gbs=alg[kd] / ms / 1e6, frac=alg[kd] / ms / 1e6 / hbm)
        out.append(rec)
    print(json.dumps({"config": cfg_name, "hbm_peak_gbs": hbm, "kernels": out}))
    print(f"\n| kernel | ms (ncu) | algorithmic | achieved | roofline frac | DRAM bytes / algorithmic |")
    print("|---|---|---|---|---|---|")
    for r in out:
        if "tflops" in r:
            extra = (f" (3xTF32 peak = bf16/6); hi/lo operands {r['operand_bytes'] / 1e6:.0f} MB at "
                     f"{r['operand_frac']:.2f} of HBM" if "operand_bytes" in r else " of burst")
            print(f"| {r['kind']} {r['which']} | {r['ms']:.3f} | {2.0 * rows * H * F / 1e12:.2f} TFLOP | "
                  f"{r['tflops']:.0f} TF/s | {r['frac_burst']:.2f}{extra} | {r['dram_bytes'] / r['alg_bytes']:.1f}x |")
        elif "gbs" in r:
            print(f"| {r['kind']} | {r['ms']:.3f} | {r['alg_bytes'] / 1e6:.0f} MB | {r['gbs']:.0f} GB/s | "
                  f"{r['frac']:.2f} of HBM | {r['dram_bytes'] / r['alg_bytes']:.2f}x |")
        else:
            print(f"| {r['kind']} ({r['kernel']}) | {r['ms']:.3f} | - | - | - | - |")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["run", "report"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--csv", default="")
    a = ap.parse_args()
    if a.mode == "run":
        run(a.config)
    else:
        report(a.config, a.csv)


if __name__ == "__main__":
    main()
