"""Device kernels through the C-ABI vs the oracle / an fp32 reference (GPU only)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from paper_2510_19470_b200 import sr as srmod
from paper_2510_19470_b200._lib import HEP_BF16, HEP_F32, check, lib
from tests import sr_golden
from tests.tolerances import F32_GEMM_MAX

pytestmark = pytest.mark.gpu


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _groups(rows, slots):
    starts = np.concatenate([[0], np.cumsum(rows)[:-1]]).astype(np.int32)
    return (torch.tensor(starts, dtype=torch.int32, device="cuda"),
            torch.tensor(np.asarray(rows, np.int32), device="cuda"),
            torch.tensor(np.asarray(slots, np.int32), device="cuda"))


def _gemm(dtype, A, B, n_slots, N, K, rows, slots, relu, sched=0):
    R = A.shape[0]
    Cout = torch.full((R, N), float("nan"), dtype=A.dtype, device="cuda")
    gs, gr, gl = _groups(rows, slots)
    check(lib.hep_grouped_gemm(dtype, A.data_ptr(), R, B.data_ptr(), n_slots, Cout.data_ptr(), N, K,
                               gs.data_ptr(), gr.data_ptr(), gl.data_ptr(), len(rows), relu, sched, _stream()))
    torch.cuda.synchronize()
    return Cout


def _reference(A, B, N, rows, slots, relu):
    out = []
    start = 0
    for r, s in zip(rows, slots):
        a = A[start:start + r].double()
        b = B[s * N:(s + 1) * N].double()
        y = a @ b.T
        out.append(torch.relu(y) if relu else y)
        start += r
    return torch.cat(out) if out else None


@pytest.mark.parametrize("pair", ["1", "0"], ids=["cta_pair", "single_cta"])
@pytest.mark.parametrize("K,N,rows,relu", [
    (256, 512, [300, 0, 128, 1, 77], 1),
    (1408, 2048, [129, 256], 0),      # cfg4 down-projection K, N multiple of 256
    (2048, 1408, [200, 513], 1),      # cfg4 up-projection: N tail (1408 = 5.5 x 256)
    (4096, 768, [1000], 0),
    (512, 1088, [300, 40], 1),        # 64-column tail: N=128 MMA on the CTA pair
    (256, 160, [70, 300], 0),         # N below one tile
])
def test_grouped_gemm_bf16(K, N, rows, relu, pair, monkeypatch):
    monkeypatch.setenv("HEP_GEMM_2CTA", pair)
    g = torch.Generator(device="cuda").manual_seed(1)
    n_slots = 3
    R = sum(rows)
    A = (torch.randn(R, K, generator=g, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(n_slots * N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    slots = [i % n_slots for i in range(len(rows))]
    got = _gemm(HEP_BF16, A, B, n_slots, N, K, rows, slots, relu).double()
    ref = _reference(A, B, N, rows, slots, relu)
    # tolerance: bf16 output rounding (2^-8 relative) + fp32 accumulation
    err = (got - ref).abs()
    tol = 2 ** -8 * ref.abs() + 1e-3 * ref.abs().max()
    assert torch.isfinite(got).all()
    assert (err <= tol).all(), f"max err {err.max().item()}"


# The headline (cfg3) shapes under the schedules the layer picks for them: the
# up-projection K=4096 -> N=14336 (A evict_last, m-fastest, 0x2) and the down-projection
# K=14336 -> N=4096, whose 117 MB per-expert A stripe takes the super-row raster of 8
# m-tiles (0x822, gemm_schedule).  Group sizes give 16, 6 and 11 m-tiles of 256 rows:
# full super-rows, a lone partial super-row and a full one followed by a partial one.
CFG3_ROWS = [4096, 1500, 2800]


@pytest.mark.parametrize("K,N,sched,relu", [
    (14336, 4096, 0x822, 0),   # cfg3 down-projection, super-row raster
    (14336, 4096, 0, 0),       # sched 0 = the layer's own pick for this shape (0x822 at 4096 rows/expert)
    (4096, 14336, 0x2, 1),     # cfg3 up-projection
    (4096, 14336, 0x822, 1),   # up-projection under the super-row raster (partial rows, N tail none)
], ids=["down_0x822", "down_auto", "up_0x2", "up_0x822"])
def test_grouped_gemm_bf16_cfg3_shapes(K, N, sched, relu):
    g = torch.Generator(device="cuda").manual_seed(3)
    n_slots = 3
    rows = CFG3_ROWS
    R = sum(rows)
    A = (torch.randn(R, K, generator=g, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(n_slots * N, K, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    slots = [2, 0, 1]
    got = _gemm(HEP_BF16, A, B, n_slots, N, K, rows, slots, relu, sched=sched)
    assert torch.isfinite(got).all()
    start = 0
    for r, sl in zip(rows, slots):  # fp64 reference, one group at a time (bounded memory)
        ref = A[start:start + r].double() @ B[sl * N:(sl + 1) * N].double().T
        if relu:
            ref = torch.relu(ref)
        err = (got[start:start + r].double() - ref).abs()
        tol = 2 ** -8 * ref.abs() + 1e-3 * ref.abs().max()
        assert (err <= tol).all(), f"group rows {r}: max err {err.max().item()}"
        start += r
    del A, B, got
    torch.cuda.empty_cache()


@pytest.mark.parametrize("K,N,rows", [(1024, 4096, [130, 0, 512]), (4096, 1024, [257, 31])])
@pytest.mark.parametrize("kernel", ["tf32x3", "simt"])
def test_grouped_gemm_f32(K, N, rows, kernel, monkeypatch):
    """fp32 grouped GEMM: the 3xTF32 tcgen05 kernel the layer ships (default; within the
    north_star's 1e-4 relative of the fp64 result on full-mantissa operands -- the dropped
    lo*lo term and fp32 TMEM accumulation) and the SIMT FFMA kernel behind
    HEP_F32_GEMM=simt (1e-5)."""
    if kernel == "simt":
        monkeypatch.setenv("HEP_F32_GEMM", "simt")
    else:
        monkeypatch.delenv("HEP_F32_GEMM", raising=False)
    g = torch.Generator(device="cuda").manual_seed(2)
    n_slots = 2
    R = sum(rows)
    A = torch.randn(R, K, generator=g, device="cuda")
    B = torch.randn(n_slots * N, K, generator=g, device="cuda") * 0.03
    slots = [i % n_slots for i in range(len(rows))]
    got = _gemm(HEP_F32, A, B, n_slots, N, K, rows, slots, 1).double()
    ref = _reference(A, B, N, rows, slots, 1)
    rel = (got - ref).abs().max() / ref.abs().max()
    assert rel < (1e-5 if kernel == "simt" else F32_GEMM_MAX), rel


@pytest.mark.parametrize("K,N,rows", [(1024, 4096, [130, 0, 512]), (4096, 1024, [257, 31]), (64, 96, [5, 300])])
def test_tf32_raw_b_split_in_smem_bitexact(K, N, rows, monkeypatch):
    """The 3xTF32 GEMM's raw-B variant (HEP_TF32_RAWB=1) streams raw fp32 B and splits it
    into hi/lo in shared memory; its products must be bit-identical to the default
    pre-split hi/lo weights (the same rna_tf32 split done by a separate kernel)."""
    monkeypatch.delenv("HEP_F32_GEMM", raising=False)
    g = torch.Generator(device="cuda").manual_seed(5)
    n_slots = 2
    A = torch.randn(sum(rows), K, generator=g, device="cuda")
    B = torch.randn(n_slots * N, K, generator=g, device="cuda") * 0.03
    slots = [(i + 1) % n_slots for i in range(len(rows))]
    monkeypatch.setenv("HEP_TF32_RAWB", "1")
    raw = _gemm(HEP_F32, A, B, n_slots, N, K, rows, slots, 1)
    monkeypatch.delenv("HEP_TF32_RAWB", raising=False)
    pre = _gemm(HEP_F32, A, B, n_slots, N, K, rows, slots, 1)
    assert torch.equal(raw, pre)


@pytest.mark.parametrize("variant", [{"HEP_GEMM_DYN": "1"}, {"HEP_GEMM_STAGES": "4"}, {"HEP_GEMM_STAGES": "6"}],
                         ids=["dynamic_tiles", "stages4", "stages6_direct"])
@pytest.mark.parametrize("K,N,rows,sched", [(1408, 2048, [129, 256, 1000], 0x6), (4096, 1408, [513, 2000], 0x822)])
def test_grouped_gemm_bf16_pair_variants_bitexact(K, N, rows, sched, variant, monkeypatch):
    """The CTA pair's opt-in variants (dynamic tile queue, 4 / 6 stages with the direct
    epilogue) run the same MMAs over the same K order per tile: outputs bit-identical to
    the default 5-stage static schedule."""
    monkeypatch.setenv("HEP_GEMM_2CTA", "1")
    g = torch.Generator(device="cuda").manual_seed(4)
    n_slots = 2
    A = (torch.randn(sum(rows), K, generator=g, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(n_slots * N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    slots = [i % n_slots for i in range(len(rows))]
    for key in ("HEP_GEMM_DYN", "HEP_GEMM_STAGES"):
        monkeypatch.delenv(key, raising=False)
    base = _gemm(HEP_BF16, A, B, n_slots, N, K, rows, slots, 1, sched=sched)
    for key, val in variant.items():
        monkeypatch.setenv(key, val)
    got = _gemm(HEP_BF16, A, B, n_slots, N, K, rows, slots, 1, sched=sched)
    assert torch.equal(got, base)


def _demo_expert_pair(h, m, seed, quantize=False):
    rng = np.random.default_rng(seed)
    P = 2 * h * m
    base = (0.05 + 0.95 * rng.random(P)) * np.where(rng.random(P) < 0.5, -1, 1)
    e = (base + rng.uniform(-0.05, 0.05, P)).astype(np.float32)
    s = base.astype(np.float32)
    if quantize:  # heavy ties in |r|
        e = (s + np.round(rng.uniform(-4, 4, P)) / 64).astype(np.float32)
    return e, s


# every select path of the encoder: sampled bracket on the cluster or the multi-block
# path, forced full-range select, and a forced invalid bracket on either path
SELECT_PATHS = ["auto", "full", "fallback", "multiblock", "fallback-multiblock"]


@pytest.mark.parametrize("h,m,ratio,k,iw,vw,per_matrix,quant", [
    (16, 24, None, 40, 32, 32, False, False),
    (16, 24, None, 40, 64, 64, False, True),
    (32, 8, None, 100, 32, 64, True, True),
    (64, 96, 50.0, None, 32, 32, False, False),
    (64, 96, 50.0, None, 32, 32, True, False),
    (8, 8, None, 0, 32, 32, False, False),
    (8, 8, None, 10 ** 9, 32, 32, False, False),
    (333, 77, 7.0, None, 64, 32, False, True),
])
@pytest.mark.parametrize("select", SELECT_PATHS)
def test_sr_encode_decode_bitexact(h, m, ratio, k, iw, vw, per_matrix, quant, select, monkeypatch):
    monkeypatch.setenv("HEP_SR_SELECT", select)
    e, s = _demo_expert_pair(h, m, seed=h * 1000 + m, quantize=quant)
    want = oracle.sr_encode(e, s, h, m, ratio=ratio, k=k, iw=iw, vw=vw, per_matrix=per_matrix,
                            use_ref=oracle.ref is not None)
    cfg = srmod.CompressionConfig(ratio_CR=ratio, k=k, index_width_bits=iw, value_width_bits=vw,
                                  per_matrix_budget=per_matrix)
    et, st = torch.from_numpy(e).cuda(), torch.from_numpy(s).cuda()
    wire = srmod.sr_encode(et, st, h, m, cfg)
    torch.cuda.synchronize()
    got = wire.cpu().numpy()
    assert got.tobytes() == want.tobytes(), "SRC1 wire differs from the reference"
    dec = srmod.sr_decode(wire, st, h, m).cpu().numpy()
    rc, want_dec = oracle.sr_decode(want, s, h, m, use_ref=oracle.ref is not None)
    assert rc == 0
    assert dec.tobytes() == want_dec.tobytes(), "decoded expert differs from the reference"


@pytest.mark.parametrize("select", ["auto", "full", "fallback", "multiblock"])
def test_sr_gpu_reference_golden_wire(select, monkeypatch):
    """The device encoder against the reference's own golden bytes
    (test_sparsecomp.cpp:258-279) -- no oracle involved."""
    monkeypatch.setenv("HEP_SR_SELECT", select)
    e = torch.from_numpy(sr_golden.REF_TEST_EXPERT).cuda()
    s = torch.from_numpy(sr_golden.REF_TEST_SHARED).cuda()
    wire = srmod.sr_encode(e, s, 1, 2, srmod.CompressionConfig(k=2))
    assert wire.cpu().numpy().tobytes() == sr_golden.REF_TEST_WIRE
    dec = srmod.sr_decode(wire, s, 1, 2).cpu().numpy()
    assert dec.tobytes() == np.array([0.0, -1.25, 0.0, 2.0], np.float32).tobytes()


@pytest.mark.parametrize("name,c", sr_golden.cases(), ids=[n for n, _ in sr_golden.cases()])
@pytest.mark.parametrize("select", ["auto", "full", "fallback", "multiblock"])
def test_sr_gpu_reference_fixtures(name, c, select, monkeypatch):
    """The device codec against the committed reference fixtures (tests/golden/sr_cases.npz,
    written from the unmodified reference by oracle/gen_golden.py): byte-identical wires and
    bit-identical decoded experts on the GPU box, where /root/reference does not exist."""
    monkeypatch.setenv("HEP_SR_SELECT", select)
    cfg = srmod.CompressionConfig(ratio_CR=c["ratio"], k=c["k"], index_width_bits=c["iw"], value_width_bits=c["vw"],
                                  per_matrix_budget=c["per_matrix"])
    e, s = torch.from_numpy(c["expert"]).cuda(), torch.from_numpy(c["shared"]).cuda()
    wire = srmod.sr_encode(e, s, c["h"], c["m"], cfg)
    assert wire.cpu().numpy().tobytes() == c["wire"].tobytes()
    dec = srmod.sr_decode(torch.from_numpy(c["wire"]).cuda(), s, c["h"], c["m"]).cpu().numpy()
    assert dec.tobytes() == c["decoded"].tobytes()


@pytest.mark.parametrize("h,m,ratio,k,per_matrix,batch", [
    (64, 96, 50.0, None, False, 3),     # fused: the split pass applies and writes back the step
    (64, 96, 50.0, None, True, 2),      # fused, per-matrix budgets (two list ranges)
    (333, 77, 7.0, None, False, 1),     # unaligned tile starts
    (8, 8, None, 0, False, 2),          # k = 0: no list range -> the step runs as its own pass
    (8, 8, None, 10 ** 9, False, 1),    # k >= P: full range -> unfused fallback
    (2048, 1408, 50.0, None, False, 4),  # cfg4 experts
])
@pytest.mark.parametrize("select", ["auto", "fallback", "multiblock"])
def test_sr_encode_fused_with_optimizer_step(h, m, ratio, k, per_matrix, batch, select, monkeypatch):
    """hep_sr_encode_update_batch == SGD step (fmaf, one rounding) then encode: masters
    bit-identical to the oracle's step, wires byte-identical to the reference encode of
    the stepped masters, and identical to the unfused GPU step + encode."""
    monkeypatch.setenv("HEP_SR_SELECT", select)
    lr = 0.0078125 * 0.75
    masters, grads, s = [], [], None
    for i in range(batch):
        e, s = _demo_expert_pair(h, m, seed=h + m + i)
        masters.append(e)
        grads.append(np.random.default_rng(i).standard_normal(2 * h * m).astype(np.float32))
    cfg = srmod.CompressionConfig(ratio_CR=ratio, k=k, per_matrix_budget=per_matrix)
    st = torch.from_numpy(s).cuda()
    dm = [torch.from_numpy(e).cuda() for e in masters]
    dg = [torch.from_numpy(g).cuda() for g in grads]
    wires = srmod.sr_encode_update_batch(dm, dg, lr, st, h, m, cfg)
    um = [torch.from_numpy(e).cuda() for e in masters]  # unfused: step, then encode
    srmod.sgd_step_batch(um, dg, lr)
    uw = srmod.sr_encode_batch(um, st, h, m, cfg)
    torch.cuda.synchronize()
    for i in range(batch):
        want_m = oracle.sgd_step(masters[i], grads[i], lr)
        assert dm[i].cpu().numpy().tobytes() == want_m.tobytes(), "stepped master differs"
        assert um[i].cpu().numpy().tobytes() == want_m.tobytes()
        want = oracle.sr_encode(want_m, s, h, m, ratio=ratio, k=k, per_matrix=per_matrix,
                                use_ref=oracle.ref is not None)
        assert wires[i].cpu().numpy().tobytes() == want.tobytes(), "fused wire differs from the reference"
        assert uw[i].cpu().numpy().tobytes() == want.tobytes()


def test_sr_bf16_expert_upcast():
    h, m = 48, 40
    e, s = _demo_expert_pair(h, m, seed=5)
    e_bf = torch.from_numpy(e).to(torch.bfloat16)
    want = oracle.sr_encode(e_bf.float().numpy(), s, h, m, k=200)
    wire = srmod.sr_encode(e_bf.cuda(), torch.from_numpy(s).cuda(), h, m, srmod.CompressionConfig(k=200))
    assert wire.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("select", ["auto", "fallback", "multiblock"])
def test_sr_cfg4_expert_bitexact(select, monkeypatch):
    """Full cfg4 expert (H=2048, F=1408, P=5,767,168) at CR=50 against the reference."""
    monkeypatch.setenv("HEP_SR_SELECT", select)
    h, m = 2048, 1408
    e, s = _demo_expert_pair(h, m, seed=11)
    want = oracle.sr_encode(e, s, h, m, ratio=50.0, use_ref=oracle.ref is not None)
    assert want.size == 461396
    cfg = srmod.CompressionConfig(ratio_CR=50.0)
    wire = srmod.sr_encode(torch.from_numpy(e).cuda(), torch.from_numpy(s).cuda(), h, m, cfg)
    assert wire.cpu().numpy().tobytes() == want.tobytes()


def test_sr_decode_rejects_corrupt_wires():
    from paper_2510_19470_b200._lib import InvalidArgument, RuntimeFailure

    h, m = 4, 4
    e, s = _demo_expert_pair(h, m, seed=3)
    st = torch.from_numpy(s).cuda()
    good = oracle.sr_encode(e, s, h, m, k=4)
    cases = []
    bad = good.copy(); bad[3] = ord("2"); cases.append((bad, RuntimeFailure, 1))           # magic
    cases.append((good[:20].copy(), RuntimeFailure, 2))                                     # truncated header
    bad = good.copy(); bad[20] = 16; cases.append((bad, RuntimeFailure, 3))                # widths
    cases.append((good[:28 + 8 * 3].copy(), RuntimeFailure, 2))                             # truncated entries
    bad = good.copy(); bad[28:32] = np.frombuffer(np.uint32(1000).tobytes(), np.uint8); cases.append((bad, RuntimeFailure, 5))
    bad = good.copy(); bad[36:40] = bad[28:32]; cases.append((bad, RuntimeFailure, 6))      # repeated index
    for wire, exc, code in cases:
        rc, _ = oracle.sr_decode(wire, s, h, m)
        assert rc == code
        with pytest.raises(exc):
            srmod.sr_decode(torch.from_numpy(wire).cuda(), st, h, m)
    with pytest.raises(InvalidArgument):
        srmod.sr_decode(torch.from_numpy(good).cuda(), torch.zeros(2 * 5 * 4, device="cuda"), 5, 4)


def test_shared_mean_bitexact():
    rng = np.random.default_rng(7)
    h, m, n = 64, 48, 8
    experts = [rng.standard_normal(2 * h * m).astype(np.float32) for _ in range(n)]
    want = oracle.shared_mean(experts, use_ref=oracle.ref is not None, h=h, m=m)
    got = srmod.shared_mean([torch.from_numpy(x).cuda() for x in experts]).cpu().numpy()
    assert got.tobytes() == want.tobytes()


def test_transpose_convert():
    x = torch.randn(100, 260, device="cuda")
    out = torch.empty(260, 100, dtype=torch.bfloat16, device="cuda")
    check(lib.hep_transpose_convert(HEP_F32, x.data_ptr(), 100, 260, HEP_BF16, out.data_ptr(), _stream()))
    torch.cuda.synchronize()
    assert torch.equal(out, x.T.contiguous().to(torch.bfloat16))


@pytest.mark.parametrize("h,m,ratio,per_matrix,quant,bf16", [
    (512, 1536, 50.0, True, False, True),    # sampled bracket (ranges >> 32768 keys)
    (512, 1536, 50.0, False, False, False),
    (512, 1536, 20.0, True, True, False),    # ~9 distinct |r|: list overflows -> full-range fallback
    (300, 1001, 100.0, True, False, False),  # odd range start (unaligned second matrix)
])
@pytest.mark.parametrize("select", ["auto", "multiblock"])
def test_sr_encode_sampled_bracket(h, m, ratio, per_matrix, quant, bf16, select, monkeypatch):
    """Medium experts where the bracket comes from a sparse sample of each range."""
    monkeypatch.setenv("HEP_SR_SELECT", select)
    e, s = _demo_expert_pair(h, m, seed=h + m, quantize=quant)
    et = torch.from_numpy(e)
    if bf16:
        et = et.to(torch.bfloat16)
        e = et.float().numpy()
    want = oracle.sr_encode(e, s, h, m, ratio=ratio, per_matrix=per_matrix, use_ref=oracle.ref is not None)
    cfg = srmod.CompressionConfig(ratio_CR=ratio, per_matrix_budget=per_matrix)
    wire = srmod.sr_encode(et.cuda(), torch.from_numpy(s).cuda(), h, m, cfg)
    assert wire.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("per_matrix", [False, True])
@pytest.mark.parametrize("select", SELECT_PATHS)
def test_sr_batched_encode_decode_bitexact(per_matrix, select, monkeypatch):
    """One launch sequence for several experts (the layer encodes all owned experts at once)."""
    monkeypatch.setenv("HEP_SR_SELECT", select)
    h, m, n = 40, 56, 5
    s = _demo_expert_pair(h, m, seed=99)[1]
    experts = [_demo_expert_pair(h, m, seed=100 + i, quantize=bool(i % 2))[0] for i in range(n)]
    cfg = srmod.CompressionConfig(ratio_CR=9.0, per_matrix_budget=per_matrix)
    st = torch.from_numpy(s).cuda()
    wires = srmod.sr_encode_batch([torch.from_numpy(e).cuda() for e in experts], st, h, m, cfg)
    outs = srmod.sr_decode_batch(wires, st, h, m)
    for e, w, o in zip(experts, wires, outs):
        want = oracle.sr_encode(e, s, h, m, ratio=9.0, per_matrix=per_matrix)
        assert w.cpu().numpy().tobytes() == want.tobytes()
        rc, dec = oracle.sr_decode(want, s, h, m)
        assert rc == 0 and o.cpu().numpy().tobytes() == dec.tobytes()
