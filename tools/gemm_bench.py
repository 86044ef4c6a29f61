"""cfg3 expert-GEMM shapes through hep_grouped_gemm (8 experts x 4096 rows): up
(K=4096 -> N=14336, ReLU) and down (K=14336 -> N=4096) under schedule words, timed with
CUDA events (median of `--reps` after warm-up, each launch alone; plus the mean of a
back-to-back burst of up+down pairs).  HEP_GEMM_STAGES / HEP_GEMM_2CTA select the variant.

    python tools/gemm_bench.py --sched-up 2 --sched-down 822,2,12,422
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
    ap.add_argument("--sched-up", default="2")
    ap.add_argument("--sched-down", default="822")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    E, R, H, F = 8, 4096, 4096, 14336
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.randn(E * R, H, generator=g, device="cuda") * 0.5).to(torch.bfloat16)
    wu = (torch.randn(E * F, H, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    wd = (torch.randn(E * H, F, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    h = torch.empty(E * R, F, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(E * R, H, dtype=torch.bfloat16, device="cuda")
    starts = torch.tensor([i * R for i in range(E)], dtype=torch.int32, device="cuda")
    rows = torch.full((E,), R, dtype=torch.int32, device="cuda")
    slots = torch.arange(E, dtype=torch.int32, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    flops = 2.0 * E * R * H * F

    def up(sched):
        check(lib.hep_grouped_gemm(HEP_BF16, x.data_ptr(), E * R, wu.data_ptr(), E, h.data_ptr(), F, H,
                                   starts.data_ptr(), rows.data_ptr(), slots.data_ptr(), E, 1, sched, st))

    def down(sched):
        check(lib.hep_grouped_gemm(HEP_BF16, h.data_ptr(), E * R, wd.data_ptr(), E, y.data_ptr(), H, F,
                                   starts.data_ptr(), rows.data_ptr(), slots.data_ptr(), E, 0, sched, st))

    def t(fn):
        ts = []
        for i in range(a.reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    env = {k: os.environ.get(k) for k in ("HEP_GEMM_STAGES", "HEP_GEMM_2CTA")}
    for su in a.sched_up.split(","):
        s_up = int(su, 16)
        ms = t(lambda: up(s_up))
        print(json.dumps({"proj": "up", "sched": hex(s_up), "ms": ms, "tflops": flops / ms / 1e9, "env": env}), flush=True)
    for sd in a.sched_down.split(","):
        s_dn = int(sd, 16)
        ms = t(lambda: down(s_dn))
        print(json.dumps({"proj": "down", "sched": hex(s_dn), "ms": ms, "tflops": flops / ms / 1e9, "env": env}),
              flush=True)
    # back-to-back pairs (the step's regime: clocks settle under the power cap)
    s_up, s_dn = int(a.sched_up.split(",")[0], 16), int(a.sched_down.split(",")[0], 16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        up(s_up), down(s_dn)
    e0.record()
    for _ in range(20):
        up(s_up)
        down(s_dn)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(json.dumps({"proj": "pair x20", "ms": ms, "tflops": 2 * flops / ms / 1e9, "env": env}), flush=True)


if __name__ == "__main__":
    main()
