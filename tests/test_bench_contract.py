"""bench.py output contract (CPU): the reference arm runs here and prints one JSON line
with the keys the driver reads; the committed round-end bench lines (profiles/r1_final/)
carry every key of the contract (value, e2e with copy bytes, roofline with its peak and
fraction, cpu_baseline, clocks sampled in the timed region, gpu_launches)."""
import glob
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(path):
    return [json.loads(ln) for ln in open(path) if ln.startswith("{")]


def test_reference_arm_prints_contract_line():
    """The reference arm prints the contract line without loading libhep.so or
    initialising CUDA (its inputs are generated on the CPU)."""
    probe = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'cfg1', '--steps', '1', "
             "'--warmup', '0']; runpy.run_path('bench.py', run_name='__main__'); import torch; "
             "maps = open('/proc/self/maps').read(); "
             "print('LOADED_LIBHEP' if 'libhep.so' in maps else 'NO_LIBHEP', "
             "'CUDA_INIT' if torch.cuda.is_initialized() else 'NO_CUDA_INIT')")
    r = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "NO_LIBHEP NO_CUDA_INIT", r.stdout[-500:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["metric"] == "MoE-layer tokens/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["higher_is_better"] is True


FINAL = sorted(glob.glob(os.path.join(ROOT, "profiles", "r1_final", "cfg*_n*.log")))


@pytest.mark.parametrize("path", FINAL, ids=[os.path.basename(p) for p in FINAL])
def test_committed_bench_line_has_contract_keys(path):
    lines = [d for d in _json_lines(path) if d.get("metric")]
    assert len(lines) == 1
    d = lines[0]
    for key in ("value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches"):
        assert key in d, key
    assert d["warmup"] >= 3 and d["scaling"] == "weak" and d["unit"] == "tokens/s"
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    roof = d["roofline"]
    assert roof["bound"] == "tensor" and roof["unit"] == "TFLOP/s"
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    assert d["clocks"]["samples"] > 0
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(d["clocks"]["reasons"])
    if d["n_gpus"] == 1:
        assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.parametrize("cfg", ["cfg1", "cfg3", "cfg4"])
def test_kernel_roofline_report_from_committed_launch_list(cfg):
    """The per-kernel roofline tables in profiles/ are reproducible from the committed ncu
    launch lists: every HBM-bound kernel of the forward at a fraction in (0, 1.05]."""
    csv = os.path.join(ROOT, "profiles", f"r1_kernel_launches_{cfg}.csv")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "kernel_roofline.py"), "report", "--config", cfg,
                        "--csv", csv], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    rep = json.loads(r.stdout.splitlines()[0])
    kinds = {k["kind"] for k in rep["kernels"]}
    assert {"K1 gate", "K2 permute", "K8 grouped GEMM", "K9 combine"} <= kinds
    for k in rep["kernels"]:
        if "frac" in k:
            assert 0 < k["frac"] <= 1.05, k
        if k["kind"] == "K8 grouped GEMM":
            assert k["tflops"] > 0
