"""3xTF32 raw-B variants: accuracy vs fp64 of each converter mode (HEP_TF32_CONV /
HEP_TF32_PRESPLIT are read once per process, so run one mode per process)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from test_gpu_kernels import _gemm, _reference, HEP_F32  # noqa: E402

res = {"mode": os.environ.get("HEP_TF32_CONV", "4"), "presplit": os.environ.get("HEP_TF32_PRESPLIT", "0")}
for K, N, rows in [(1024, 4096, [128] * 8), (4096, 1024, [128] * 8)]:
    g = torch.Generator(device="cuda").manual_seed(7)
    A = torch.randn(sum(rows), K, generator=g, device="cuda")
    B = torch.randn(8 * N, K, generator=g, device="cuda") * 0.03
    slots = list(range(8))
    got = _gemm(HEP_F32, A, B, 8, N, K, rows, slots, 0).double()
    ref = _reference(A, B, N, rows, slots, 0)
    res[f"K{K}_N{N}_maxrel"] = ((got - ref).abs().max() / ref.abs().max()).item()
    res[f"K{K}_N{N}_meanrel"] = ((got - ref).abs().mean() / ref.abs().max()).item()
print(json.dumps(res))
