"""SR encode of a batch of cfg4 experts (the per-rank owned experts at N=2 / N=4: 32 / 16)
timed as a CUDA-graph replay, for per-kernel ncu captures of the encode chain.

    python tools/sr_encode_probe.py [--batch 16] [--reps 20]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_2510_19470_b200 import sr  # noqa: E402
from bench_sr import timed  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    h, m = 2048, 1408
    P = 2 * h * m
    g = torch.Generator(device="cuda").manual_seed(0)
    base = (0.05 + 0.95 * torch.rand(P, generator=g, device="cuda")) * \
        (torch.randint(0, 2, (P,), generator=g, device="cuda") * 2 - 1)
    shared = base.float()
    experts = [(base + (torch.rand(P, generator=g, device="cuda") * 2 - 1) * 0.05).float() for _ in range(a.batch)]
    cfg = sr.CompressionConfig(ratio_CR=50.0)
    t = timed(lambda: sr.sr_encode_batch(experts, shared, h, m, cfg), a.reps)
    print(json.dumps({"shape": "cfg4", "batch": a.batch, "encode_batch_ms": t,
                      "gbs": a.batch * 2 * P * 4 / t / 1e6}), flush=True)


if __name__ == "__main__":
    main()
