"""The C++ step API (include/hybridep/moe.hpp: RAII Communicator / Layer over the C-ABI,
rethrowing std::domain_error / std::invalid_argument / std::runtime_error like the
reference, plus resolve_plan / write_plan_reports) driven by a plain C++ program,
tests/cpp/test_moe_api.cpp, built by `make -C paper_2510_19470_b200/csrc cpp-test`."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "csrc", "test_moe_api")


def _build():
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2510_19470_b200", "csrc"), "-s", "cpp-test"], check=True)


def test_cpp_api_host_checks():
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "C++ API checks passed" in r.stdout


@pytest.mark.gpu
def test_cpp_api_forward_matches_oracle(tmp_path):
    import oracle
    from tests import tolerances as tol

    _build()
    r = subprocess.run([BIN, "gpu", str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr

    def bf(name, shape):
        u = np.fromfile(tmp_path / name, np.uint16).astype(np.uint32) << 16
        return u.view(np.float32).reshape(shape)

    H, F, E, k, T = 256, 512, 8, 2, 50
    x, wg = bf("x.bin", (T, H)), bf("wg.bin", (H, E))
    up, down, y = bf("up.bin", (E, H, F)), bf("down.bin", (E, F, H)), bf("y.bin", (T, H))
    ref = oracle.moe_layer(x[None], wg, up, down, k, [1], [1], bf16=True)
    scale = np.abs(ref["y"][0]).max()
    d = np.abs(y - ref["y"][0])
    assert d.max() <= tol.BF16_VS_MIRROR_MAX * scale and d.mean() <= tol.BF16_VS_MIRROR_MEAN * scale
