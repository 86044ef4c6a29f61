"""SREncode fused with the optimizer step vs the two passes (PAPER.md:1185 claims -30%):
per expert shape, time hep_sgd_step_batch + hep_sr_encode_batch against
hep_sr_encode_update_batch (CUDA events, median of 20 after 3 warm-ups).  Algorithmic
bytes of the step+encode: read master, grad, shared, write master (16 B/element) + wire.

    python tools/bench_sr_fused.py > gpurun_out/sr_fused.log
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_19470_b200 import sr as srmod  # noqa: E402


def timeit(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    for name, h, m, batch in [("cfg4", 2048, 1408, 8), ("cfg1", 1024, 4096, 1), ("cfg3", 4096, 14336, 1)]:
        P = 2 * h * m
        g = torch.Generator(device="cuda").manual_seed(1)
        base = (0.05 + 0.95 * torch.rand(P, generator=g, device="cuda")) * (torch.randint(0, 2, (P,), generator=g, device="cuda") * 2 - 1)
        shared = base.float()
        masters = [(base + (torch.rand(P, generator=g, device="cuda") * 2 - 1) * 0.05).float() for _ in range(batch)]
        grads = [torch.randn(P, generator=g, device="cuda") * 1e-3 for _ in range(batch)]
        cfg = srmod.CompressionConfig(ratio_CR=50.0)
        lr = 1e-3
        unfused = timeit(lambda: (srmod.sgd_step_batch(masters, grads, lr), srmod.sr_encode_batch(masters, shared, h, m, cfg)))
        step_only = timeit(lambda: srmod.sgd_step_batch(masters, grads, lr))
        fused = timeit(lambda: srmod.sr_encode_update_batch(masters, grads, lr, shared, h, m, cfg))
        alg = batch * (16 * P + srmod.wire_bytes(h, m, cfg))
        print(json.dumps({"shape": name, "h": h, "m": m, "batch": batch, "unfused_ms": unfused, "sgd_only_ms": step_only,
                          "fused_ms": fused, "saving": 1 - fused / unfused,
                          "fused_gbs": alg / (fused / 1e3) / 1e9,
                          "fused_hbm_frac": alg / (fused / 1e3) / 1e9 / peaks["hbm_gbs"]}), flush=True)


if __name__ == "__main__":
    main()
