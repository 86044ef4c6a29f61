"""Full MoE-layer step through the C-ABI vs the CPU oracle (GPU only).

Routing (top-k indices), the permutation (pos) and per-(dest, expert) counts must be
bit-exact; outputs within the stated tolerance:
  * fp32 layers: max |y - y_ref| <= 1e-4 * max |y_ref|   (north_star: 1e-4 relative)
  * bf16 layers: tests/tolerances.py BF16_VS_MIRROR_* against the oracle that mirrors the
    bf16 rounding points of h, y_expert and y (the remaining difference is fp32-vs-fp64
    accumulation flipping a bf16 rounding); accuracy against the fp32 reference is stated
    in tests/test_gpu_headline.py
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2510_19470_b200 import synthetic
from paper_2510_19470_b200 import InvalidArgument
from paper_2510_19470_b200.moe import MoELayer
from tests import tolerances as tol

pytestmark = pytest.mark.gpu


def run_layer(H, F, E, k, T, dtype, seed=0, gaussian=False):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn((T, H), generator=g).to(dtype) if gaussian else synthetic.dyadic((T, H), g, dtype=dtype)
    wg = synthetic.dyadic((H, E), g)
    w_up, w_down = synthetic.experts(E, H, F, g, dtype=dtype)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=dtype)
    layer.set_gate(wg.cuda())
    for e in range(E):
        layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
    y = layer.forward(x.cuda())
    dbg = layer.debug(T)
    torch.cuda.synchronize()
    ref = oracle.moe_layer(x.float().numpy()[None], wg.numpy(), w_up.float().numpy(), w_down.float().numpy(), k,
                           [1], [1], bf16=dtype == torch.bfloat16)
    layer.close()
    return x, y.float().cpu().numpy(), dbg, ref


def check_routing(dbg, ref):
    assert np.array_equal(dbg["topk_idx"].cpu().numpy(), ref["topk_idx"][0])
    np.testing.assert_allclose(dbg["topk_w"].cpu().numpy(), ref["topk_w"][0], rtol=2e-6, atol=1e-7)
    assert np.array_equal(dbg["pos"].cpu().numpy(), ref["pos"][0])
    assert np.array_equal(dbg["key_counts"].cpu().numpy(), ref["key_counts"][0])


def check_packed(x, dbg, k):
    # packed[pos[t, j]] == x[t]
    packed = dbg["packed"].float().cpu()
    pos = dbg["pos"].cpu().long()
    for j in range(k):
        assert torch.equal(packed[pos[:, j]], x.float())


def test_layer_fp32_cfg1_shape():
    """cfg1 per-GPU shape (H=1024, F=4096, E=8, k=2, T=512, fp32)."""
    x, y, dbg, ref = run_layer(1024, 4096, 8, 2, 512, torch.float32)
    check_routing(dbg, ref)
    check_packed(x, dbg, 2)
    err = np.abs(y - ref["y"][0]).max() / np.abs(ref["y"][0]).max()
    assert err <= tol.F32_MAX, err


def test_layer_fp32_gaussian_inputs():
    """fp32 accuracy on full-mantissa activations (N(0,1) tokens: the 3xTF32 split of x
    has a non-zero lo part, unlike dyadic inputs): max error <= 1e-4 of max |y|."""
    x, y, dbg, ref = run_layer(1024, 4096, 8, 2, 512, torch.float32, seed=5, gaussian=True)
    assert np.array_equal(dbg["topk_idx"].cpu().numpy(), ref["topk_idx"][0])
    err = np.abs(y - ref["y"][0]).max() / np.abs(ref["y"][0]).max()
    assert err <= tol.F32_MAX, err


def test_layer_bf16_small_ragged():
    x, y, dbg, ref = run_layer(512, 1024, 8, 2, 1000, torch.bfloat16, seed=3)
    check_routing(dbg, ref)
    check_packed(x, dbg, 2)
    scale = np.abs(ref["y"][0]).max()
    d = np.abs(y - ref["y"][0])
    assert d.max() <= tol.BF16_VS_MIRROR_MAX * scale and d.mean() <= tol.BF16_VS_MIRROR_MEAN * scale, \
        (d.max() / scale, d.mean() / scale)


def test_layer_bf16_cfg4_shape():
    """cfg4 expert shape (H=2048, F=1408, E=64, k=6) at G=1, T=256."""
    x, y, dbg, ref = run_layer(2048, 1408, 64, 6, 256, torch.bfloat16, seed=4)
    check_routing(dbg, ref)
    scale = np.abs(ref["y"][0]).max()
    d = np.abs(y - ref["y"][0])
    assert d.max() <= tol.BF16_VS_MIRROR_MAX * scale and d.mean() <= tol.BF16_VS_MIRROR_MEAN * scale, \
        (d.max() / scale, d.mean() / scale)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
def test_layer_single_token_empty_and_repeat(dtype):
    """Edge cases: T=1, an empty batch (T=0: no rows, an empty result, state intact), and
    further forwards on the same layer reusing its buffers."""
    H, F, E, k = 256, 512, 8, 2
    bf16 = dtype == torch.bfloat16
    g = torch.Generator().manual_seed(9)
    wg = synthetic.dyadic((H, E), g)
    w_up, w_down = synthetic.experts(E, H, F, g, dtype=dtype)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=64, dtype=dtype)
    layer.set_gate(wg.cuda())
    for e in range(E):
        layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
    for T in (1, 0, 64, 0, 33):
        x = synthetic.dyadic((T, H), g, dtype=dtype)
        y = layer.forward(x.cuda())
        yh = torch.empty(T, H, dtype=dtype).pin_memory()
        layer.forward_host(x.pin_memory(), yh)
        layer.host_fence()
        torch.cuda.synchronize()
        assert tuple(y.shape) == (T, H) and tuple(yh.shape) == (T, H)
        if T == 0:
            continue
        y = y.float().cpu().numpy()
        ref = oracle.moe_layer(x.float().numpy()[None], wg.numpy(), w_up.float().numpy(), w_down.float().numpy(),
                               k, [1], [1], bf16=bf16)
        scale = np.abs(ref["y"][0]).max()
        assert np.abs(y - ref["y"][0]).max() <= (tol.BF16_VS_MIRROR_MAX if bf16 else tol.F32_MAX) * scale
        assert np.array_equal(yh.float().numpy(), y)
    with pytest.raises(InvalidArgument):
        layer.forward(torch.zeros(65, H, dtype=dtype, device="cuda"))
    layer.close()


def test_layer_forward_host_matches_device():
    H, F, E, k, T = 256, 512, 8, 2, 100
    g = torch.Generator().manual_seed(10)
    x = synthetic.dyadic((T, H), g, dtype=torch.bfloat16)
    wg = synthetic.dyadic((H, E), g)
    w_up, w_down = synthetic.experts(E, H, F, g, dtype=torch.bfloat16)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=torch.bfloat16)
    layer.set_gate(wg.cuda())
    for e in range(E):
        layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
    y_dev = layer.forward(x.cuda()).cpu()
    xh = x.pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    layer.forward_host(xh, yh)
    torch.cuda.synchronize()
    assert torch.equal(y_dev, yh)
    layer.close()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_refresh_shared_single_gpu(dtype):
    """refresh_shared with every expert local: the mean over the owned fp32 masters,
    bit-exact with the reference's init_shared (sparsecomp.cpp:147-168)."""
    from paper_2510_19470_b200.sr import CompressionConfig

    H, F, E = 128, 192, 8
    g = torch.Generator().manual_seed(3)
    w_up, w_down = synthetic.experts(E, H, F, g, dtype=dtype)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=2, max_tokens=64, dtype=dtype,
                     sr=CompressionConfig(ratio_CR=8.0))
    for e in range(E):
        layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
    layer.refresh_shared()
    got = layer.get_shared().cpu().numpy()
    flat = [torch.cat([w_up[e].float().reshape(-1), w_down[e].float().reshape(-1)]).numpy() for e in range(E)]
    assert got.tobytes() == oracle.shared_mean(flat).tobytes()
    layer.close()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
def test_layer_graph_replay_matches_eager(dtype):
    """One-GPU layers replay the step as a CUDA graph per (x, T, y).  Replays must equal the
    eager step (profiled forwards run eagerly) bit for bit, see new data written into the
    same x buffer, and follow weight updates."""
    H, F, E, k, T = 256, 512, 8, 2, 100
    g = torch.Generator().manual_seed(21)
    wg = synthetic.dyadic((H, E), g)
    w_up, w_down = synthetic.experts(E, H, F, g, dtype=dtype)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=dtype)
    layer.set_gate(wg.cuda())
    for e in range(E):
        layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
    x = synthetic.dyadic((T, H), g, dtype=dtype).cuda()
    y = torch.empty_like(x)
    side = torch.cuda.Stream()
    for stream in (None, side):  # the legacy default stream and a side stream
        outs = []
        for _ in range(3):  # capture, then replays
            layer.forward(x, out=y, stream=stream)
            torch.cuda.synchronize()
            outs.append(y.clone())
        layer.set_profiling(2)
        layer.forward(x, out=y, stream=stream)  # eager
        torch.cuda.synchronize()
        layer.timings()
        layer.set_profiling(0)
        for o in outs:
            assert torch.equal(o, y)
    x2 = synthetic.dyadic((T, H), g, dtype=dtype).cuda()
    x.copy_(x2)  # same buffer, new tokens: the replay reads them
    layer.forward(x, out=y)
    torch.cuda.synchronize()
    ref = oracle.moe_layer(x2.float().cpu().numpy()[None], wg.numpy(), w_up.float().numpy(), w_down.float().numpy(), k,
                           [1], [1], bf16=dtype == torch.bfloat16)
    scale = np.abs(ref["y"][0]).max()
    assert np.abs(y.float().cpu().numpy() - ref["y"][0]).max() <= (
        tol.BF16_VS_MIRROR_MAX if dtype == torch.bfloat16 else tol.F32_MAX) * scale
    layer.set_expert(0, (w_up[0] * 2).cuda(), w_down[0].cuda())  # weights change -> new result
    layer.forward(x, out=y)
    torch.cuda.synchronize()
    w_up2 = w_up.clone()
    w_up2[0] *= 2
    ref2 = oracle.moe_layer(x2.float().cpu().numpy()[None], wg.numpy(), w_up2.float().numpy(), w_down.float().numpy(),
                            k, [1], [1], bf16=dtype == torch.bfloat16)
    assert np.abs(y.float().cpu().numpy() - ref2["y"][0]).max() <= (
        tol.BF16_VS_MIRROR_MAX if dtype == torch.bfloat16 else tol.F32_MAX) * np.abs(ref2["y"][0]).max()
    layer.close()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
def test_layer_residual_form(dtype):
    """hep_layer_forward_residual: y = x + MoE(x) with the add fused into the combine,
    against the fp32 reference + x (bf16: tests/tolerances.py BF16_VS_FP32_*)."""
    H, F, E, k, T = 512, 1024, 8, 2, 300
    g = torch.Generator().manual_seed(23)
    x = synthetic.dyadic((T, H), g, dtype=dtype)
    wg = synthetic.dyadic((H, E), g)
    w_up, w_down = synthetic.experts(E, H, F, g, dtype=dtype)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=dtype)
    layer.set_gate(wg.cuda())
    for e in range(E):
        layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
    y = layer.forward(x.cuda(), residual=True).float().cpu().numpy()
    torch.cuda.synchronize()
    layer.close()
    bf16 = dtype == torch.bfloat16
    ref = oracle.moe_layer(x.float().numpy()[None], wg.numpy(), w_up.float().numpy(), w_down.float().numpy(), k, [1],
                           [1], bf16=bf16, exact=bf16)
    want = ref["y"][0] + x.float().numpy()
    m, mean = tol.rel_errors(y, want)
    if bf16:
        assert m <= tol.BF16_VS_FP32_MAX and mean <= tol.BF16_VS_FP32_MEAN, (m, mean)
    else:
        assert m <= tol.F32_MAX, m


@pytest.mark.parametrize("H,F,E,k,T", [(512, 1024, 8, 2, 1000), (2048, 1408, 64, 6, 777), (256, 512, 8, 2, 1)])
def test_gathered_a_matches_permuted_bitexact(H, F, E, k, T, monkeypatch):
    """HEP_GATHER_A=1 (one GPU) fuses the permute into the up-projection's A load (x rows
    gathered by the inverse routing map).  Against the explicit permute the GEMM inputs
    are the same bf16 rows in the same order, so y must be bit-identical --
    ragged groups, partial m-tiles, top-6 and a single token included; the inspection
    path still reproduces the packed rows."""
    g = torch.Generator().manual_seed(11)
    x = torch.randn((T, H), generator=g).to(torch.bfloat16).cuda()
    wg = torch.randn((H, E), generator=g) * 0.05
    w_up, w_down = synthetic.experts(E, H, F, g, dtype=torch.bfloat16)
    outs = []
    for gather in ("1", "0"):
        monkeypatch.setenv("HEP_GATHER_A", gather)
        layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=torch.bfloat16)
        layer.set_gate(wg.cuda())
        for e in range(E):
            layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
        y = layer.forward(x)
        y2 = layer.forward(x)  # second step: the inverse map is rewritten, not accumulated
        dbg = layer.debug(T)
        torch.cuda.synchronize()
        check_packed(x.cpu(), dbg, k)
        outs.append((y.clone(), y2.clone()))
        layer.close()
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    assert torch.equal(outs[0][0], outs[0][1])


def test_fp32_layer_raw_weights_bitexact(monkeypatch):
    """fp32 layer with HEP_TF32_RAWB=1 (the 3xTF32 GEMMs stream the raw fp32 compute
    copies and split them in shared memory) vs the default pre-split hi/lo weights: the
    same rna split feeds the same MMAs, so y is bit-identical."""
    H, F, E, k, T = 1024, 4096, 8, 2, 300
    g = torch.Generator().manual_seed(21)
    x = torch.randn((T, H), generator=g).cuda()
    wg = torch.randn((H, E), generator=g) * 0.05
    w_up, w_down = synthetic.experts(E, H, F, g, dtype=torch.float32)
    outs = []
    for raw in ("1", "0"):
        monkeypatch.setenv("HEP_TF32_RAWB", raw)
        layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=torch.float32)
        layer.set_gate(wg.cuda())
        for e in range(E):
            layer.set_expert(e, w_up[e].cuda(), w_down[e].cuda())
        outs.append(layer.forward(x).clone())
        torch.cuda.synchronize()
        layer.close()
    assert torch.equal(outs[0], outs[1])
