"""Interleaved A/B timing of cfg3 down-/up-projection GEMM variants (schedule word x
HEP_GEMM_STAGES), so clock drift under the power cap does not bias the comparison: every
round runs every variant (3 launches, median), rounds repeat; reports the median over
rounds per variant.

    python tools/gemm_ab.py --proj down --variants 822:5,822:6,422:5,822:4 --rounds 6
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_19470_b200._lib import HEP_BF16, check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--proj", default="down")
    ap.add_argument("--variants", default="822:5,822:6,422:5,822:4")
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--data", default="layer", help="layer: dyadic tokens + demo experts (the bench's); randn")
    a = ap.parse_args()
    E, R, H, F = 8, 4096, 4096, 14336
    g = torch.Generator(device="cuda").manual_seed(0)
    if a.data == "randn":
        x = (torch.randn(E * R, H, generator=g, device="cuda") * 0.5).to(torch.bfloat16)
        wu = (torch.randn(E * F, H, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
        wd = (torch.randn(E * H, F, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    else:
        x = (torch.randint(-8, 9, (E * R, H), generator=g, device="cuda").float() / 16).to(torch.bfloat16)
        base = (0.05 + 0.95 * torch.rand(F, H, generator=g, device="cuda")) * (torch.randint(0, 2, (F, H), generator=g, device="cuda") * 2 - 1)
        wu = torch.cat([((base + (torch.rand(F, H, generator=g, device="cuda") * 2 - 1) * 0.05) / 64) for _ in range(E)]).to(torch.bfloat16)
        based = (0.05 + 0.95 * torch.rand(H, F, generator=g, device="cuda")) * (torch.randint(0, 2, (H, F), generator=g, device="cuda") * 2 - 1)
        wd = torch.cat([((based + (torch.rand(H, F, generator=g, device="cuda") * 2 - 1) * 0.05) / 64) for _ in range(E)]).to(torch.bfloat16)
    h = torch.empty(E * R, F, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(E * R, H, dtype=torch.bfloat16, device="cuda")
    starts = torch.tensor([i * R for i in range(E)], dtype=torch.int32, device="cuda")
    rows = torch.full((E,), R, dtype=torch.int32, device="cuda")
    slots = torch.arange(E, dtype=torch.int32, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    flops = 2.0 * E * R * H * F

    def run(proj, sched):
        if proj == "up":
            check(lib.hep_grouped_gemm(HEP_BF16, x.data_ptr(), E * R, wu.data_ptr(), E, h.data_ptr(), F, H,
                                       starts.data_ptr(), rows.data_ptr(), slots.data_ptr(), E, 1, sched, st))
        else:
            check(lib.hep_grouped_gemm(HEP_BF16, h.data_ptr(), E * R, wd.data_ptr(), E, y.data_ptr(), H, F,
                                       starts.data_ptr(), rows.data_ptr(), slots.data_ptr(), E, 0, sched, st))

    run("up", 0x2)  # h = relu(x w_up): the down-projection's real A operand
    torch.cuda.synchronize()
    # sched:stages[:dyn]
    variants = [(int(v.split(":")[0], 16), v.split(":")[1], v.split(":")[2] if v.count(":") > 1 else "1")
                for v in a.variants.split(",")]
    res = {v: [] for v in variants}
    for _ in range(a.rounds):
        for v in variants:
            os.environ["HEP_GEMM_STAGES"] = v[1]
            os.environ["HEP_GEMM_DYN"] = v[2]
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run(a.proj, v[0])
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[v].append(statistics.median(ts))
    for v in variants:
        ms = statistics.median(res[v])
        print(json.dumps({"proj": a.proj, "sched": hex(v[0]), "stages": v[1], "dyn": v[2], "ms": ms, "tflops": flops / ms / 1e9,
                          "rounds_ms": [round(t, 3) for t in res[v]], "data": a.data}), flush=True)


if __name__ == "__main__":
    main()
