"""Synthetic inputs of the named shapes (no datasets or checkpoints exist offline).

Distributions follow SURVEY.md §8(d):
  * tokens x and gate W_g: dyadic values {-8..8}/16, so every fp32 partial sum of a
    logit is exact and routing is independent of summation order (bit-exact top-k);
  * experts: the reference demo population (cli_app.cpp:89-118): a base matrix with
    |v| in [0.05, 1] and random sign, plus U(-noise, noise) per expert, scaled by a
    power of two (2^-5 at H <= 1024, 2^-6 above) so the scaling is exact.
"""
from __future__ import annotations

import torch


def expert_scale(hidden: int) -> float:
    return 2.0 ** -5 if hidden <= 1024 else 2.0 ** -6


def dyadic(shape, gen: torch.Generator, device="cpu", dtype=torch.float32) -> torch.Tensor:
    v = torch.randint(-8, 9, shape, generator=gen, device=device, dtype=torch.int32)
    return (v.to(torch.float32) / 16.0).to(dtype)


def experts(E: int, H: int, F: int, gen: torch.Generator, device="cpu", dtype=torch.float32, noise=0.05):
    """Returns (w_up [E,H,F], w_down [E,F,H]) in `dtype` (values exactly representable)."""
    s = expert_scale(H)

    def base(shape):
        mag = 0.05 + 0.95 * torch.rand(shape, generator=gen, device=device, dtype=torch.float64)
        sign = torch.randint(0, 2, shape, generator=gen, device=device) * 2 - 1
        return mag * sign

    bu, bd = base((H, F)), base((F, H))
    ups, downs = [], []
    for _ in range(E):
        nu = (torch.rand((H, F), generator=gen, device=device, dtype=torch.float64) * 2 - 1) * noise
        nd = (torch.rand((F, H), generator=gen, device=device, dtype=torch.float64) * 2 - 1) * noise
        ups.append(((bu + nu).to(torch.float32) * s).to(dtype))
        downs.append(((bd + nd).to(torch.float32) * s).to(dtype))
    return torch.stack(ups), torch.stack(downs)
