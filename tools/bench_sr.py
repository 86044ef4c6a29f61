"""Migration codec (K5 encode / K6 decode / K7 shared mean) on one B200, per expert shape
of BASELINE configs, against the HBM roofline, with the reference's own single-thread
CPU codec (oracle/_ref, compiled from /root/reference) timed beside it.

    python tools/bench_sr.py [--reps 20] [--shapes cfg1,cfg4,cfg3]

Algorithmic bytes: encode 2*P*b_in read + (28 + 8k) written; decode
P*4 (shared) + (28 + 8k) read + P*4 written; shared mean E*P*b read + P*4 written.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_19470_b200 import sr  # noqa: E402

SHAPES = {"cfg1": (1024, 4096, 8), "cfg4": (2048, 1408, 64), "cfg3": (4096, 14336, 8)}


def timed(fn, reps):
    """Device time per call: the call is captured once in a CUDA graph and replayed, so
    host-side Python/ctypes overhead (tens of us) does not leak into small-expert timings."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--shapes", default="cfg1,cfg4,cfg3")
    ap.add_argument("--cpu", action="store_true", help="also time the reference CPU codec")
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    hbm = peaks["hbm_gbs"]
    out = []
    for name in a.shapes.split(","):
        h, m, E = SHAPES[name]
        P = 2 * h * m
        g = torch.Generator(device="cuda").manual_seed(0)
        base = (0.05 + 0.95 * torch.rand(P, generator=g, device="cuda")) * \
            (torch.randint(0, 2, (P,), generator=g, device="cuda") * 2 - 1)
        expert = (base + (torch.rand(P, generator=g, device="cuda") * 2 - 1) * 0.05).float()
        shared = base.float()
        cfg = sr.CompressionConfig(ratio_CR=50.0)
        k = cfg.resolve_k(P)
        wire = sr.sr_encode(expert, shared, h, m, cfg)
        t_enc = timed(lambda: sr.sr_encode(expert, shared, h, m, cfg), a.reps)
        t_dec = timed(lambda: sr.sr_decode(wire, shared, h, m, check_status=False), a.reps)
        nb = min(E, 8)  # experts owned per GPU at G=8 (cfg4) / all experts (cfg1, cfg3)
        batch = [expert + float(i) * 2 ** -12 for i in range(nb)]
        t_enc_b = timed(lambda: sr.sr_encode_batch(batch, shared, h, m, cfg), max(2, a.reps // 4))
        wires_b = sr.sr_encode_batch(batch, shared, h, m, cfg)
        t_dec_b = timed(lambda: sr.sr_decode_batch(wires_b, shared, h, m, check_status=False), max(2, a.reps // 4))
        n_mean = min(E, 8)
        experts = [expert + float(i) * 2 ** -10 for i in range(n_mean)]  # distinct buffers (no L2 reuse)
        t_mean = timed(lambda: sr.shared_mean(experts), a.reps)
        wb = 28 + 8 * k
        rec = {"shape": name, "h": h, "m": m, "P": P, "k": k, "wire_bytes": wb,
               "encode_ms": t_enc, "encode_gbs": (2 * P * 4 + wb) / t_enc / 1e6,
               "decode_ms": t_dec, "decode_gbs": (P * 4 + wb + P * 4) / t_dec / 1e6,
               "shared_mean_ms": t_mean, "shared_mean_experts": n_mean,
               "shared_mean_gbs": (n_mean * P * 4 + P * 4) / t_mean / 1e6, "hbm_peak_gbs": hbm}
        rec.update(batch=nb, encode_batch_ms=t_enc_b, encode_batch_gbs=nb * (2 * P * 4 + wb) / t_enc_b / 1e6,
                   decode_batch_ms=t_dec_b, decode_batch_gbs=nb * (2 * P * 4 + wb) / t_dec_b / 1e6)
        rec["encode_batch_frac"] = rec["encode_batch_gbs"] / hbm
        rec["decode_batch_frac"] = rec["decode_batch_gbs"] / hbm
        rec["encode_frac"] = rec["encode_gbs"] / hbm
        rec["decode_frac"] = rec["decode_gbs"] / hbm
        rec["shared_mean_frac"] = rec["shared_mean_gbs"] / hbm
        if a.cpu:
            import oracle
            if oracle.ref is not None:
                e_np, s_np = expert.cpu().numpy(), shared.cpu().numpy()
                t0 = time.perf_counter()
                w_np = oracle.sr_encode(e_np, s_np, h, m, ratio=50.0, use_ref=True)
                rec["ref_cpu_encode_s"] = time.perf_counter() - t0
                t0 = time.perf_counter()
                oracle.sr_decode(w_np, s_np, h, m, use_ref=True)
                rec["ref_cpu_decode_s"] = time.perf_counter() - t0
                rec["wire_equal_ref"] = bool(w_np.tobytes() == wire.cpu().numpy().tobytes())
        out.append(rec)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
