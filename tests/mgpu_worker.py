"""Multi-GPU parity worker (one process per GPU, launched by tests/test_gpu_multi.py via
torch.distributed.run).  Every rank builds the same global synthetic problem, runs its
share through the C-ABI (NCCL inside libhep.so) and checks it against the CPU oracle
executed over the same G simulated GPUs:
  * routing (top-k ids), permutation (pos) and per-(dest, expert) counts bit-exact;
  * outputs within the bf16 / fp32 tolerances of tests/test_gpu_layer.py;
  * --sr: experts migrate as SR wires; the expected output uses the decoded expert
    wherever the computing GPU is not the owner (oracle decode, bit-exact with the GPU).
"""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before torch creates the context

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2510_19470_b200 import synthetic  # noqa: E402
from paper_2510_19470_b200 import topology as topo  # noqa: E402
from paper_2510_19470_b200.moe import Communicator, MoELayer  # noqa: E402
from paper_2510_19470_b200.sr import CompressionConfig  # noqa: E402
from tests import tolerances as tol  # noqa: E402


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
    ap.add_argument("--ragged", action="store_true",
                    help="every rank a different token count (down to 1), then a second forward "
                         "with the counts rotated and a third with rank 0 empty, reusing the "
                         "layer's buffers")
    ap.add_argument("--out", default="")
    a = ap.parse_args()

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = Communicator.from_torch()
    G = int(np.prod(a.sf))
    assert G == world
    bf16 = a.dtype == "bf16"
    dt = torch.bfloat16 if bf16 else torch.float32

    g = torch.Generator().manual_seed(42)
    x_all = synthetic.dyadic((G, a.T, a.H), g, dtype=dt)
    wg = synthetic.dyadic((a.H, a.E), g)
    w_up, w_down = synthetic.experts(a.E, a.H, a.F, g, dtype=dt)

    sr = CompressionConfig(ratio_CR=8.0) if a.sr else None
    layer = MoELayer(hidden=a.H, ffn=a.F, experts=a.E, top_k=a.k, max_tokens=a.T, dtype=dt, sf=a.sf, sed=a.sed,
                     rank=rank, comm=comm, sr=sr)
    layer.set_gate(wg.cuda())
    P = 2 * a.H * a.F
    flat = [torch.cat([w_up[e].float().reshape(-1), w_down[e].float().reshape(-1)]).numpy() for e in range(a.E)]
    shared = oracle.shared_mean(flat)
    for e in layer.owned_experts():
        layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
    if a.sr:
        # the shared expert from every rank's owned experts (cross-GPU chain), twice: the
        # second refresh must reuse the partial buffers safely and give the same bytes
        for _ in range(2):
            layer.refresh_shared()
            got = layer.get_shared().cpu().numpy()
            assert got.tobytes() == shared.tobytes(), "refreshed shared expert differs from the reference mean"
    layer.gather_experts()
    if a.ragged:
        counts = [max(1, a.T - 113 * r) for r in range(G)]
        counts[-1] = 1
        zero = list(counts)
        zero[0] = 0  # an empty batch on rank 0: it still serves its peers' rows
        plan = [counts, counts[1:] + counts[:1], zero]
    else:
        plan = [[a.T] * G]
    report = {"rank": rank, "sf": a.sf, "sed": a.sed, "sr": a.sr, "T": [c[rank] for c in plan]}
    for counts in plan:
        check(a, layer, x_all[:, :counts[rank]], wg, w_up, w_down, flat, shared, rank, G, bf16, report)
    if a.out and rank == 0:
        json.dump(report, open(a.out, "w"))
    print("rank", rank, "ok", report, flush=True)
    layer.close()
    comm.close()
    dist.destroy_process_group()


def check(a, layer, x_all, wg, w_up, w_down, flat, shared, rank, G, bf16, report):
    """One forward of this rank's x_all[rank] against the oracle.  Rows of other ranks
    beyond their own count are never routed, so x_all[:, :T_rank] gives the oracle
    exactly this rank's tokens and routing."""
    T = x_all.shape[1]
    y = layer.forward(x_all[rank].cuda())
    torch.cuda.synchronize()
    verify(a, layer, y, x_all, wg, w_up, w_down, flat, shared, rank, G, bf16, report)


def verify(a, layer, y, x_all, wg, w_up, w_down, flat, shared, rank, G, bf16, report):
    """This rank's finished forward (y on the device) against the oracle over G
    simulated GPUs (also used by tests/vrank_worker.py for virtual ranks)."""
    T = x_all.shape[1]
    if T == 0:
        assert tuple(y.shape) == (0, a.H)
        return
    dbg = layer.debug(T)
    y = y.float().cpu().numpy()
    if not a.sr:
        ref = oracle.moe_layer(x_all.float().numpy(), wg.numpy(), w_up.float().numpy(), w_down.float().numpy(),
                               a.k, a.sf, a.sed, bf16=bf16)
        assert np.array_equal(dbg["topk_idx"].cpu().numpy(), ref["topk_idx"][rank]), "top-k differs"
        assert np.array_equal(dbg["pos"].cpu().numpy(), ref["pos"][rank]), "permutation differs"
        assert np.array_equal(dbg["key_counts"].cpu().numpy(), ref["key_counts"][rank]), "counts differ"
        want = ref["y"][rank]
    else:
        # Weights as seen by the GPU that computes each (token, expert): exact at the
        # owner, SR-decoded anywhere else (decode is bit-exact with the oracle's).
        route = topo.route_table(topo.ClusterSpec.of(a.sf, a.sed))
        n = a.E // G
        up_eff = w_up.float().numpy().copy()
        down_eff = w_down.float().numpy().copy()
        HF = a.H * a.F
        for e in range(a.E):
            o = e // n
            if route[rank, o] != o:
                wire = oracle.sr_encode(flat[e], shared, a.H, a.F, ratio=8.0)
                rc, dec = oracle.sr_decode(wire, shared, a.H, a.F)
                assert rc == 0
                if bf16:
                    dec = torch.from_numpy(dec).to(torch.bfloat16).float().numpy()
                up_eff[e] = dec[:HF].reshape(a.H, a.F)
                down_eff[e] = dec[HF:].reshape(a.F, a.H)
        ref = oracle.moe_layer(x_all[rank:rank + 1].float().numpy(), wg.numpy(), up_eff, down_eff, a.k, [1], [1],
                               bf16=bf16)
        assert np.array_equal(dbg["topk_idx"].cpu().numpy(), ref["topk_idx"][0]), "top-k differs"
        want = ref["y"][0]
    scale = float(np.abs(want).max())
    d = np.abs(y - want)
    report.update(max_rel=float(d.max() / scale), mean_rel=float(d.mean() / scale))
    if bf16:
        assert d.max() <= tol.BF16_VS_MIRROR_MAX * scale and d.mean() <= tol.BF16_VS_MIRROR_MEAN * scale, report
    else:
        assert d.max() <= tol.F32_MAX * scale, report


if __name__ == "__main__":
    main()
