"""Virtual-rank parity worker: ONE process drives all G ranks of a hierarchy on ONE GPU
(hep_comm_init_virtual), every rank on its own stream, through the peer-memory step the
multi-GPU path runs -- device-side count exchange, dispatch stores into the peers'
receive areas, the GEMM epilogue's stores back into the sources' output buffers,
epoch flags, expert All-Gather pulls (dense or SR wires) and the shared-expert chain.
Launched by tests/test_gpu_vranks.py (one subprocess per case, under a timeout).

Checks per rank (tests/mgpu_worker.verify): routing, permutation and counts bit-exact
with the oracle over G simulated GPUs, outputs within tests/tolerances.py; the SR
shared-expert refresh bit-exact with the reference mean.  Options:
  --ragged   different token counts per rank, rotated, then rank 0 empty
  --update   new expert weights between two steps (the All-Gather slot-4 guard)
  --corrupt  SR: corrupt one gathered wire; the layer must raise RuntimeFailure
  --mismatch rank 1 with a different max_tokens: the first step must raise InvalidArgument
  --sgd      SR: an SGD step fused with the migration encode (hep_layer_sgd_step) between
             two steps; the second must match the oracle on the stepped experts
"""
import argparse
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before torch creates the context
os.environ.setdefault("HEP_P2P_TIMEOUT_S", "60")  # a lost flag traps with a diagnostic

import numpy as np  # noqa: E402
import torch  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import oracle  # noqa: E402
from mgpu_worker import verify  # noqa: E402
from paper_2510_19470_b200 import InvalidArgument, RuntimeFailure, synthetic  # noqa: E402
from paper_2510_19470_b200.moe import Communicator, MoELayer  # noqa: E402
from paper_2510_19470_b200.sr import CompressionConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=int, nargs="+", required=True)
    ap.add_argument("--sed", type=int, nargs="+", required=True)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--H", type=int, default=256)
    ap.add_argument("--F", type=int, default=512)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--T", type=int, default=300)
    ap.add_argument("--sr", action="store_true")
    ap.add_argument("--ragged", action="store_true")
    ap.add_argument("--update", action="store_true")
    ap.add_argument("--corrupt", action="store_true")
    ap.add_argument("--mismatch", action="store_true")
    ap.add_argument("--sgd", action="store_true")
    ap.add_argument("--residual", action="store_true",
                    help="also run the residual form y = x + MoE(x) and check it against the plain step + x")
    ap.add_argument("--dump", default="", help="save every rank's first-step output (bf16 bits) to this .npy")
    a = ap.parse_args()

    torch.cuda.set_device(0)
    G = int(np.prod(a.sf))
    bf16 = a.dtype == "bf16"
    dt = torch.bfloat16 if bf16 else torch.float32
    g = torch.Generator().manual_seed(42)
    x_all = synthetic.dyadic((G, a.T, a.H), g, dtype=dt)
    wg = synthetic.dyadic((a.H, a.E), g)
    w_up, w_down = synthetic.experts(a.E, a.H, a.F, g, dtype=dt)

    comms = Communicator.virtual(G)
    streams = [torch.cuda.Stream() for _ in range(G)]
    sr = CompressionConfig(ratio_CR=8.0) if a.sr else None
    layers = []
    for r in range(G):
        tmax = a.T + 8 if (a.mismatch and r == 1) else a.T
        layers.append(MoELayer(hidden=a.H, ffn=a.F, experts=a.E, top_k=a.k, max_tokens=tmax, dtype=dt, sf=a.sf,
                               sed=a.sed, rank=r, comm=comms[r], sr=sr))
    if a.mismatch:
        with torch.cuda.stream(streams[0]):
            try:
                layers[0].forward(x_all[0].cuda())
            except InvalidArgument as e:
                assert "different shape" in str(e), e
                print("mismatch rejected:", e, flush=True)
            else:
                raise AssertionError("a rank with a different max_tokens was not rejected")
        for L in layers:
            L.close()
        return

    def each(fn):
        for r in range(G):
            with torch.cuda.stream(streams[r]):
                fn(r, layers[r])

    def load(w_up, w_down):
        flat = [torch.cat([w_up[e].float().reshape(-1), w_down[e].float().reshape(-1)]).numpy() for e in range(a.E)]
        wg_d = wg.cuda()
        each(lambda r, L: L.set_gate(wg_d, stream=streams[r]))
        each(lambda r, L: [L.set_expert(e, w_up[e].cuda(), w_down[e].cuda(), stream=streams[r])
                           for e in L.owned_experts()])
        shared = oracle.shared_mean(flat)
        if a.sr:
            # the cross-rank chain twice: the second refresh reuses the partials safely
            for _ in range(2):
                each(lambda r, L: L.refresh_shared(stream=streams[r]))
                torch.cuda.synchronize()
                for L in layers:
                    got = L.get_shared().cpu().numpy()
                    assert got.tobytes() == shared.tobytes(), "refreshed shared expert differs from the reference mean"
        each(lambda r, L: L.gather_experts(stream=streams[r]))
        return flat, shared

    flat, shared = load(w_up, w_down)

    if a.corrupt:
        assert a.sr
        layers[0].debug_corrupt_next_gather()
        each(lambda r, L: L.gather_experts(stream=streams[r]))
        # the rejection surfaces at the first call after the failed decode completed (the
        # rank's share of that collective step is still enqueued, so no peer hangs) or at
        # check(), whichever comes first
        errors = []
        for r in range(G):
            with torch.cuda.stream(streams[r]):
                try:
                    layers[r].forward(x_all[r].cuda(), stream=streams[r])
                except RuntimeFailure as e:
                    errors.append((r, str(e)))
        torch.cuda.synchronize()
        try:
            layers[0].check()
        except RuntimeFailure as e:
            errors.append((0, str(e)))
        assert [r for r, _ in errors] == [0], errors
        assert "bad residual magic" in errors[0][1], errors
        print("corrupt wire rejected:", errors[0][1], flush=True)
        for r in range(1, G):
            layers[r].check()  # the other ranks decoded clean wires
        # the next gather re-encodes: the layer works again
        each(lambda r, L: L.gather_experts(stream=streams[r]))

    if a.ragged:
        counts = [max(1, a.T - 113 * r) for r in range(G)]
        counts[-1] = 1
        zero = list(counts)
        zero[0] = 0
        plan = [counts, counts[1:] + counts[:1], zero]
    else:
        plan = [[a.T] * G]

    def step(counts, w_up, w_down, flat, shared):
        xs = x_all[:, :max(counts)] if len(set(counts)) == 1 else None
        ys = [None] * G
        for r in range(G):
            with torch.cuda.stream(streams[r]):
                ys[r] = layers[r].forward(x_all[r, :counts[r]].cuda(), stream=streams[r])
        torch.cuda.synchronize()
        if a.dump and not getattr(step, "dumped", False):
            np.save(a.dump, np.stack([y.view(torch.int16).cpu().numpy() if y.dtype == torch.bfloat16
                                      else y.view(torch.int32).cpu().numpy() for y in ys]))
            step.dumped = True
        for r in range(G):
            report = {"rank": r, "T": counts[r]}
            xr = x_all[:, :counts[r]] if xs is None else xs
            verify(a, layers[r], ys[r], xr, wg, w_up, w_down, flat, shared, r, G, bf16, report)
            print("rank", r, "ok", report, flush=True)

    for counts in plan:
        step(counts, w_up, w_down, flat, shared)
    if a.residual:
        plain, res = [None] * G, [None] * G
        xs = [x_all[r].cuda() for r in range(G)]
        for r in range(G):
            with torch.cuda.stream(streams[r]):
                plain[r] = layers[r].forward(xs[r], stream=streams[r])
        for r in range(G):
            with torch.cuda.stream(streams[r]):
                res[r] = layers[r].forward(xs[r], stream=streams[r], residual=True)
        torch.cuda.synchronize()
        for r in range(G):
            want = xs[r].double() + plain[r].double()
            d = (res[r].double() - want).abs()
            # one rounding of x + sum vs the plain step's rounding of the sum
            bound = (2.0 ** -8 if bf16 else 2.0 ** -22) * (plain[r].double().abs() + res[r].double().abs()) + 1e-30
            assert bool((d <= bound).all()), (r, float(d.max()))
        print("residual ok", flush=True)
    if a.sgd:
        assert a.sr
        lr = 2.0 ** -7
        rng = np.random.default_rng(7)
        grads = [rng.standard_normal(2 * a.H * a.F).astype(np.float32) * 2.0 ** -6 for _ in range(a.E)]
        for r in range(G):
            with torch.cuda.stream(streams[r]):
                layers[r].sgd_step([torch.from_numpy(grads[e]).cuda() for e in layers[r].owned_experts()], lr,
                                   stream=streams[r])
        each(lambda r, L: L.gather_experts(stream=streams[r]))
        flat2 = [oracle.sgd_step(flat[e], grads[e], lr) for e in range(a.E)]
        HF = a.H * a.F
        # what an owner computes with: its stepped master in the layer dtype
        w_up2 = torch.stack([torch.from_numpy(f[:HF].reshape(a.H, a.F)) for f in flat2]).to(dt)
        w_down2 = torch.stack([torch.from_numpy(f[HF:].reshape(a.F, a.H)) for f in flat2]).to(dt)
        step(plan[0], w_up2, w_down2, flat2, shared)
        print("sgd ok", flush=True)
    if a.update:
        # new weights on every owner between steps: peers must not pull torn experts
        g2 = torch.Generator().manual_seed(4242)
        w_up2, w_down2 = synthetic.experts(a.E, a.H, a.F, g2, dtype=dt)
        flat2, shared2 = load(w_up2, w_down2)
        step(plan[0], w_up2, w_down2, flat2, shared2)
        print("update ok", flush=True)
    for L in layers:
        L.check()
        L.close()
    for c in comms:
        c.close()


if __name__ == "__main__":
    main()
