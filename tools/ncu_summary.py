"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv>          # per-kernel launch list
    python tools/ncu_summary.py full <report.ncu-rep>            # key metrics per captured kernel
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict, defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ni = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi or r[ni] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("hep::<unnamed>::", "").replace("(anonymous namespace)::", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    out = {k: {"launches": len(v), "mean_us": sum(v) / len(v) / 1e3, "share": sum(v) / total}
           for k, v in agg.items()}
    return out


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if mode == "launches" else full(path), indent=1))
