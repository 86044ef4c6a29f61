"""Routing parity of every rank of an 8-GPU hierarchy on ONE GPU (hep_route_plan):
cfg2's S_ED sweep (fp32, SF=[2,4]) and cfg4's 3-level hierarchy (bf16, E=64, k=6).
Top-k ids, the packed-buffer permutation and the per-(dest, expert) counts must be
bit-exact with the CPU oracle run over 8 simulated GPUs; plus cfg1 end to end."""
import ctypes as C
import itertools

import numpy as np
import pytest
import torch

import oracle
from paper_2510_19470_b200 import synthetic
from paper_2510_19470_b200._lib import HEP_BF16, HEP_F32, Level, check, lib
from paper_2510_19470_b200.moe import MoELayer

pytestmark = pytest.mark.gpu


def route_plan(sf, sed, rank, x, wg, k):
    T, H = x.shape
    E = wg.shape[1]
    G = int(np.prod(sf))
    lv = (Level * len(sf))(*[Level(a, b, 1e9) for a, b in zip(sf, sed)])
    ti = torch.empty(T * k, dtype=torch.int32, device="cuda")
    tw = torch.empty(T * k, dtype=torch.float32, device="cuda")
    pos = torch.empty(T * k, dtype=torch.int32, device="cuda")
    kc = torch.empty(G * E, dtype=torch.int32, device="cuda")
    dt = HEP_BF16 if x.dtype == torch.bfloat16 else HEP_F32
    check(lib.hep_route_plan(lv, len(sf), rank, dt, x.data_ptr(), T, H, wg.data_ptr(), E, k, ti.data_ptr(),
                             tw.data_ptr(), pos.data_ptr(), kc.data_ptr(),
                             C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return ti.view(T, k).cpu().numpy(), tw.view(T, k).cpu().numpy(), pos.view(T, k).cpu().numpy(), kc.cpu().numpy()


def check_hierarchy(sf, sed, x_all, wg, k, bf16):
    G, T, H = x_all.shape
    E = wg.shape[1]
    F = 64  # routing does not depend on the FFN
    w_up = np.zeros((E, H, F), np.float32)
    w_down = np.zeros((E, F, H), np.float32)
    ref = oracle.moe_layer(x_all.float().numpy(), wg.float().numpy(), w_up, w_down, k, sf, sed, bf16=bf16,
                           stride=T + 1)
    for r in range(G):
        ti, tw, pos, kc = route_plan(sf, sed, r, x_all[r].cuda(), wg.cuda(), k)
        assert np.array_equal(ti, ref["topk_idx"][r]), (sf, sed, r)
        assert np.array_equal(pos, ref["pos"][r]), (sf, sed, r)
        assert np.array_equal(kc, ref["key_counts"][r]), (sf, sed, r)
        np.testing.assert_allclose(tw, ref["topk_w"][r], rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("sed", [[1, 1], [1, 2], [1, 4], [2, 1], [2, 2], [2, 4]])
def test_cfg2_sed_sweep_routing_bitexact(sed):
    """cfg2: H=1024, E=8, top-2, 512 tokens on each of 8 GPUs, fp32, SF=[2,4]."""
    g = torch.Generator().manual_seed(20)
    x_all = synthetic.dyadic((8, 512, 1024), g)
    wg = synthetic.dyadic((1024, 8), g)
    check_hierarchy([2, 4], sed, x_all, wg, 2, bf16=False)


@pytest.mark.parametrize("sed", [list(s) for s in itertools.product([1, 2], repeat=3)])
def test_cfg4_hierarchy_routing_bitexact(sed):
    """cfg4: H=2048, E=64, top-6, SF=[2,2,2], every S_ED, bf16, 256 tokens per GPU."""
    g = torch.Generator().manual_seed(21)
    x_all = synthetic.dyadic((8, 256, 2048), g, dtype=torch.bfloat16)
    wg = synthetic.dyadic((2048, 64), g, dtype=torch.bfloat16)
    check_hierarchy([2, 2, 2], sed, x_all, wg, 6, bf16=True)


@pytest.mark.parametrize("gate,split", [("mma", "0"), ("umma", "1")])
@pytest.mark.parametrize("E,k,T", [(8, 2, 300), (64, 6, 200)])
def test_gate_variants_routing_bitexact(gate, split, E, k, T, monkeypatch):
    """The mma.sync gate (HEP_GATE=mma) and the K-split tcgen05 gate (HEP_GATE_SPLIT=1)
    route exactly like the default tcgen05 gate and the oracle (ragged token counts)."""
    monkeypatch.setenv("HEP_GATE", gate)
    monkeypatch.setenv("HEP_GATE_SPLIT", split)
    g = torch.Generator().manual_seed(22 + E)
    x_all = synthetic.dyadic((8, T, 1024), g, dtype=torch.bfloat16)
    wg = synthetic.dyadic((1024, E), g, dtype=torch.bfloat16)
    check_hierarchy([2, 4], [1, 2], x_all, wg, k, bf16=True)


def test_cfg1_full_layer_vs_8_simulated_gpus():
    """cfg1: 4096 tokens total (8 simulated GPUs x 512), H=1024, F=4096, E=8, top-2, fp32,
    SF=[2,4], S_ED=[1,4].  Dense experts make every GPU's output independent of where its
    rows are computed, so one B200 running all 4096 tokens must match the oracle's
    8-GPU run row for row (routing bit-exact, outputs 1e-4 relative)."""
    g = torch.Generator().manual_seed(1)
    G, T, H, F, E, k = 8, 512, 1024, 4096, 8, 2
    x_all = synthetic.dyadic((G, T, H), g)
    wg = synthetic.dyadic((H, E), g)
    w_up, w_down = synthetic.experts(E, H, F, g)
    ref = oracle.moe_layer(x_all.numpy(), wg.numpy(), w_up.numpy(), w_down.numpy(), k, [2, 4], [1, 4], bf16=False)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=G * T, dtype=torch.float32)
    layer.set_gate(wg.cuda())
    for e in range(E):
        layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
    y = layer.forward(x_all.reshape(G * T, H).cuda())
    dbg = layer.debug(G * T)
    torch.cuda.synchronize()
    assert np.array_equal(dbg["topk_idx"].cpu().numpy(), ref["topk_idx"].reshape(G * T, k))
    y = y.cpu().numpy().reshape(G, T, H)
    rel = np.abs(y - ref["y"]).max() / np.abs(ref["y"]).max()
    assert rel <= 1e-4, rel
    layer.close()
