"""The benchmarked configuration itself, bf16 accuracy against the fp32 reference, and
routing on realistic (non-dyadic) inputs (GPU only).

* cfg3 (BASELINE.json configs[2], the bench line): H=4096, F=14336, E=8, top-2, 16,384
  tokens, bf16, through the same MoELayer and the same GEMM schedules the bench runs
  (up 0x2; down 0x822, the super-row raster).  Routing, permutation and counts are
  checked bit-exact on every token; outputs on every 64th token (the oracle's FFN is
  ~60 TFLOP for all of them) against both the mirrored-rounding oracle and the fp32
  reference (tests/tolerances.py).
* Realistic routing: Gaussian tokens and a non-dyadic gate.  The device accumulates
  logits in fp32 on the tensor cores, the oracle in fp64, so an order-dependent
  near-tie may legitimately flip a choice; every disagreement must coincide with a
  logit gap below the fp32 accumulation bound, and the permutation must be exactly the
  stable counting sort of the device's own choices.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from paper_2510_19470_b200 import synthetic
from paper_2510_19470_b200._lib import HEP_BF16, Level, check, lib
from paper_2510_19470_b200.moe import MoELayer
from tests import tolerances as tol

pytestmark = pytest.mark.gpu


def _device_problem(H, F, E, k, T, seed, dtype=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = synthetic.dyadic((T, H), g, device="cuda", dtype=dtype)
    wg = synthetic.dyadic((H, E), g, device="cuda")
    w_up, w_down = synthetic.experts(E, H, F, g, device="cuda", dtype=dtype)
    return x, wg, w_up, w_down


def _stable_positions(topk_idx, E):
    """S7 at G=1: pos of (t, j) = rank of (t, j) in the stable counting sort by expert."""
    flat = topk_idx.reshape(-1).astype(np.int64)
    order = np.argsort(flat, kind="stable")
    pos = np.empty_like(flat)
    pos[order] = np.arange(flat.size)
    counts = np.bincount(flat, minlength=E)
    return pos.reshape(topk_idx.shape).astype(np.int32), counts.astype(np.int32)


def test_cfg3_headline_layer(record_accuracy):
    H, F, E, k, T, stride = 4096, 14336, 8, 2, 16384, 64
    x, wg, w_up, w_down = _device_problem(H, F, E, k, T, seed=2024)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=torch.bfloat16)
    up_sched, down_sched = layer.gemm_schedule()
    # the schedules the bench line runs: the down-projection's 117 MB per-expert A stripe
    # takes the super-row raster (gemm_sm100.cu gemm_schedule)
    assert (up_sched, down_sched) == (0x2, 0x822), (hex(up_sched), hex(down_sched))
    layer.set_gate(wg)
    for e in range(E):
        layer.set_expert(e, w_up[e], w_down[e])
    y = layer.forward(x)
    dbg = layer.debug(T)
    torch.cuda.synchronize()
    xs = x.float().cpu().numpy()[None]
    wgs = wg.cpu().numpy()
    ups = w_up.float().cpu().numpy()
    downs = w_down.float().cpu().numpy()
    del w_up, w_down
    layer.close()
    mirror = oracle.moe_layer(xs, wgs, ups, downs, k, [1], [1], bf16=True, stride=stride)
    exact = oracle.moe_layer(xs, wgs, ups, downs, k, [1], [1], bf16=True, stride=stride, exact=True)
    # routing, permutation, counts: every token, bit-exact
    assert np.array_equal(dbg["topk_idx"].cpu().numpy(), mirror["topk_idx"][0])
    np.testing.assert_allclose(dbg["topk_w"].cpu().numpy(), mirror["topk_w"][0], rtol=2e-6, atol=1e-7)
    assert np.array_equal(dbg["pos"].cpu().numpy(), mirror["pos"][0])
    assert np.array_equal(dbg["key_counts"].cpu().numpy(), mirror["key_counts"][0])
    rows = np.arange(0, T, stride)
    yg = y.float().cpu().numpy()[rows]
    m_max, m_mean = tol.rel_errors(yg, mirror["y"][0][rows])
    e_max, e_mean = tol.rel_errors(yg, exact["y"][0][rows])
    record_accuracy(config="cfg3", rows=len(rows), vs_mirror_max=m_max, vs_mirror_mean=m_mean, vs_fp32_max=e_max,
                    vs_fp32_mean=e_mean)
    assert m_max <= tol.BF16_VS_MIRROR_MAX and m_mean <= tol.BF16_VS_MIRROR_MEAN, (m_max, m_mean)
    assert e_max <= tol.BF16_VS_FP32_MAX and e_mean <= tol.BF16_VS_FP32_MEAN, (e_max, e_mean)


@pytest.mark.parametrize("H,F,E,k,T,name", [
    (2048, 1408, 64, 6, 2048, "cfg4"),
    (512, 1024, 8, 2, 1000, "small"),
    (1024, 4096, 8, 2, 512, "cfg1_bf16"),
])
def test_bf16_accuracy_vs_fp32_reference(H, F, E, k, T, name, record_accuracy):
    """bf16 layers against the fp32 reference (north_star): the oracle in exact mode."""
    x, wg, w_up, w_down = _device_problem(H, F, E, k, T, seed=H + E)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=torch.bfloat16)
    layer.set_gate(wg)
    for e in range(E):
        layer.set_expert(e, w_up[e], w_down[e])
    y = layer.forward(x).float().cpu().numpy()
    torch.cuda.synchronize()
    layer.close()
    args = (x.float().cpu().numpy()[None], wg.cpu().numpy(), w_up.float().cpu().numpy(),
            w_down.float().cpu().numpy(), k, [1], [1])
    mirror = oracle.moe_layer(*args, bf16=True)
    exact = oracle.moe_layer(*args, bf16=True, exact=True)
    m_max, m_mean = tol.rel_errors(y, mirror["y"][0])
    e_max, e_mean = tol.rel_errors(y, exact["y"][0])
    record_accuracy(config=name, rows=T, vs_mirror_max=m_max, vs_mirror_mean=m_mean, vs_fp32_max=e_max,
                    vs_fp32_mean=e_mean)
    assert m_max <= tol.BF16_VS_MIRROR_MAX and m_mean <= tol.BF16_VS_MIRROR_MEAN, (m_max, m_mean)
    assert e_max <= tol.BF16_VS_FP32_MAX and e_mean <= tol.BF16_VS_FP32_MEAN, (e_max, e_mean)


@pytest.mark.parametrize("H,E,k,T", [(4096, 8, 2, 16384), (2048, 64, 6, 16384), (1024, 8, 2, 4096)])
def test_routing_realistic_inputs_tie_margin(H, E, k, T, record_accuracy):
    g = torch.Generator(device="cuda").manual_seed(77 + E)
    x = torch.randn((T, H), generator=g, device="cuda").to(torch.bfloat16)
    wg = (torch.randn((H, E), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    lv = (Level * 1)(Level(1, 1, 1e9))
    ti = torch.empty(T * k, dtype=torch.int32, device="cuda")
    tw = torch.empty(T * k, dtype=torch.float32, device="cuda")
    pos = torch.empty(T * k, dtype=torch.int32, device="cuda")
    kc = torch.empty(E, dtype=torch.int32, device="cuda")
    check(lib.hep_route_plan(lv, 1, 0, HEP_BF16, x.data_ptr(), T, H, wg.data_ptr(), E, k, ti.data_ptr(),
                             tw.data_ptr(), pos.data_ptr(), kc.data_ptr(),
                             C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ti = ti.view(T, k).cpu().numpy()
    tw = tw.view(T, k).cpu().numpy()
    # the permutation and counts are exact functions of the device's own choices
    want_pos, want_counts = _stable_positions(ti, E)
    assert np.array_equal(pos.view(T, k).cpu().numpy(), want_pos)
    assert np.array_equal(kc.cpu().numpy(), want_counts)
    # choices vs the fp64 oracle
    xf, wf = x.float().cpu().numpy(), wg.float().cpu().numpy()
    ref_idx, ref_w = oracle.gate(xf, wf, k)
    logits = xf.astype(np.float64) @ wf.astype(np.float64)                  # exact products, fp64 sums
    # fp32 accumulation of H products (any order): |err| <= H * 2^-24 * sum |x_h w_h|, per
    # expert; a swap of two experts needs their true gap below the sum of both bounds
    bound = H * 2.0 ** -24 * (np.abs(xf).astype(np.float64) @ np.abs(wf).astype(np.float64))
    bad = np.nonzero((ti != ref_idx).any(axis=1))[0]
    for t in bad:
        for j in range(k):
            a, b = ti[t, j], ref_idx[t, j]
            if a != b:
                gap = abs(logits[t, a] - logits[t, b])
                assert gap <= bound[t, a] + bound[t, b], (t, j, a, b, gap, bound[t, a] + bound[t, b])
    same = np.setdiff1d(np.arange(T), bad)
    # weights: softmax of the selected logits; differences come from the logits' fp32
    # accumulation only
    np.testing.assert_allclose(tw[same], ref_w[same], rtol=0, atol=1e-4)
    record_accuracy(config=f"routing H={H} E={E} k={k}", tokens=T, disagreements=int(len(bad)),
                    max_w_err=float(np.abs(tw[same] - ref_w[same]).max()))
