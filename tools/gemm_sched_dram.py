"""One launch of the cfg3 down-projection GEMM per (schedule, stages) variant, for an ncu
metrics pass (DRAM bytes, duration, SM clock per launch):

    ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \\
        --clock-control none --csv python tools/gemm_sched_dram.py
"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_19470_b200._lib import HEP_BF16, check, lib  # noqa: E402

UP_VARIANTS = [(0x2, "5", "0"), (0x2, "5", "1")]
VARIANTS = [(0x822, "5", "0"), (0x822, "5", "1"), (0x2, "5", "1"), (0x422, "5", "1"), (0x822, "4", "0")]


def main():
    E, R, H, F = 8, 4096, 4096, 14336
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.relu(torch.randint(-8, 9, (E * R, F), generator=g, device="cuda").float() / 16).to(torch.bfloat16)
    base = (0.05 + 0.95 * torch.rand(H, F, generator=g, device="cuda")) * (torch.randint(0, 2, (H, F), generator=g, device="cuda") * 2 - 1)
    wd = torch.cat([((base + (torch.rand(H, F, generator=g, device="cuda") * 2 - 1) * 0.05) / 64) for _ in range(E)]).to(torch.bfloat16)
    y = torch.empty(E * R, H, dtype=torch.bfloat16, device="cuda")
    starts = torch.tensor([i * R for i in range(E)], dtype=torch.int32, device="cuda")
    rows = torch.full((E,), R, dtype=torch.int32, device="cuda")
    slots = torch.arange(E, dtype=torch.int32, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    x = (torch.randint(-8, 9, (E * R, H), generator=g, device="cuda").float() / 16).to(torch.bfloat16)
    wu = torch.cat([((torch.rand(F, H, generator=g, device="cuda") * 2 - 1) / 64) for _ in range(E)]).to(torch.bfloat16)
    hh = torch.empty(E * R, F, dtype=torch.bfloat16, device="cuda")
    for sched, stages, dyn in UP_VARIANTS:
        os.environ["HEP_GEMM_STAGES"] = stages
        os.environ["HEP_GEMM_DYN"] = dyn
        check(lib.hep_grouped_gemm(HEP_BF16, x.data_ptr(), E * R, wu.data_ptr(), E, hh.data_ptr(), F, H,
                                   starts.data_ptr(), rows.data_ptr(), slots.data_ptr(), E, 1, sched, st))
        torch.cuda.synchronize()
        print("up variant", hex(sched), "stages", stages, "dyn", dyn, flush=True)
    for sched, deep, dyn in VARIANTS:
        os.environ["HEP_GEMM_STAGES"] = deep
        os.environ["HEP_GEMM_DYN"] = dyn
        check(lib.hep_grouped_gemm(HEP_BF16, h.data_ptr(), E * R, wd.data_ptr(), E, y.data_ptr(), H, F,
                                   starts.data_ptr(), rows.data_ptr(), slots.data_ptr(), E, 0, sched, st))
        torch.cuda.synchronize()
        print("variant", hex(sched), "stages", deep, "dyn", dyn, flush=True)


if __name__ == "__main__":
    main()
