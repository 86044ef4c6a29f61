"""One encode (single expert and a batch of 8) per BASELINE expert shape, no graphs: the
command `ncu` wraps for the SR codec's launch lists (see profiles/README.md).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_sr.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_19470_b200 import sr  # noqa: E402

SHAPES = {"cfg4": (2048, 1408), "cfg3": (4096, 14336)}


def main():
    for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else SHAPES):
        h, m = SHAPES[name]
        P = 2 * h * m
        g = torch.Generator(device="cuda").manual_seed(0)
        base = (0.05 + 0.95 * torch.rand(P, generator=g, device="cuda")) * \
            (torch.randint(0, 2, (P,), generator=g, device="cuda") * 2 - 1)
        expert = (base + (torch.rand(P, generator=g, device="cuda") * 2 - 1) * 0.05).to(torch.bfloat16)
        shared = base.float()
        cfg = sr.CompressionConfig(ratio_CR=50.0)
        sr.sr_encode(expert, shared, h, m, cfg)
        batch = [(expert.float() + float(i) * 2 ** -12).to(torch.bfloat16) for i in range(8)]
        sr.sr_encode_batch(batch, shared, h, m, cfg)
        torch.cuda.synchronize()
        print(name, "ok", flush=True)


if __name__ == "__main__":
    main()
