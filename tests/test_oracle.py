"""Pins the CPU restatement (oracle/moe_oracle.c) before it is trusted as the checker
(CPU only): its SR codec against the reference's own golden wire
(test_sparsecomp.cpp:258-279) and the reference fixtures in tests/golden/sr_cases.npz,
and -- where oracle/_ref is built -- byte for byte against the reference library on
randomized cases (continuous, heavy-tie, per-matrix, 32/64-bit)."""
import numpy as np
import pytest

import oracle
from tests import sr_golden


def test_orc_reference_golden_wire():
    wire = oracle.sr_encode(sr_golden.REF_TEST_EXPERT, sr_golden.REF_TEST_SHARED, 1, 2, k=2)
    assert wire.tobytes() == sr_golden.REF_TEST_WIRE
    rc, dec = oracle.sr_decode(wire, sr_golden.REF_TEST_SHARED, 1, 2)
    # k = 2 keeps the two largest residuals: 0.5 is dropped
    assert rc == 0 and dec.tobytes() == np.array([0.0, -1.25, 0.0, 2.0], np.float32).tobytes()


@pytest.mark.parametrize("name,c", sr_golden.cases(), ids=[n for n, _ in sr_golden.cases()])
def test_orc_matches_reference_fixtures(name, c):
    wire = oracle.sr_encode(c["expert"], c["shared"], c["h"], c["m"], ratio=c["ratio"], k=c["k"], iw=c["iw"],
                            vw=c["vw"], per_matrix=c["per_matrix"])
    assert wire.tobytes() == c["wire"].tobytes()
    rc, dec = oracle.sr_decode(c["wire"], c["shared"], c["h"], c["m"])
    assert rc == 0 and dec.tobytes() == c["decoded"].tobytes()


def test_orc_rejects_corrupt_wires_like_the_reference():
    """sparsecomp.cpp:36 (magic), :113 (truncation), :236-238 (index bounds / order)."""
    wire = bytearray(sr_golden.REF_TEST_WIRE)
    s = sr_golden.REF_TEST_SHARED
    bad = bytearray(wire)
    bad[3] = ord("2")
    assert oracle.sr_decode(np.frombuffer(bytes(bad), np.uint8), s, 1, 2)[0] == 1
    assert oracle.sr_decode(np.frombuffer(bytes(wire[:-3]), np.uint8), s, 1, 2)[0] == 2
    oob = bytearray(wire)
    oob[36] = 9  # second index 3 -> 9 >= P = 4
    assert oracle.sr_decode(np.frombuffer(bytes(oob), np.uint8), s, 1, 2)[0] == 5
    order = bytearray(wire)
    order[36] = 1  # second index 3 -> 1, not increasing
    assert oracle.sr_decode(np.frombuffer(bytes(order), np.uint8), s, 1, 2)[0] == 6


@pytest.mark.skipif(oracle.ref is None, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", range(40))
def test_orc_matches_reference_library_randomized(seed):
    rng = np.random.default_rng(seed)
    h, m = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    P = 2 * h * m
    base = (0.05 + 0.95 * rng.random(P)) * np.where(rng.random(P) < 0.5, -1, 1)
    s = base.astype(np.float32)
    if seed % 3 == 0:
        e = (s + np.round(rng.uniform(-3, 3, P)) / 32).astype(np.float32)  # heavy ties in |r|
    else:
        e = (base + rng.uniform(-0.05, 0.05, P)).astype(np.float32)
    iw, vw = [(32, 32), (64, 64), (32, 64), (64, 32)][seed % 4]
    pm = bool(seed % 2)
    kw = dict(k=int(rng.integers(0, P + 3))) if seed % 5 else dict(ratio=float(rng.uniform(1.5, 60)))
    a = oracle.sr_encode(e, s, h, m, iw=iw, vw=vw, per_matrix=pm, **kw)
    b = oracle.sr_encode(e, s, h, m, iw=iw, vw=vw, per_matrix=pm, use_ref=True, **kw)
    assert a.tobytes() == b.tobytes()
    ra, da = oracle.sr_decode(a, s, h, m)
    rb, db = oracle.sr_decode(b, s, h, m, use_ref=True)
    assert ra == rb == 0 and da.tobytes() == db.tobytes()
    experts = [e, s, (e + s).astype(np.float32)]
    assert oracle.shared_mean(experts).tobytes() == oracle.shared_mean(experts, use_ref=True, h=h, m=m).tobytes()


@pytest.mark.parametrize("bf16", [False, True])
def test_batched_layer_equals_per_row_definition(bf16):
    """The oracle's layer batches the FFN per expert (weights streamed once per expert);
    every sampled token's output must equal the per-row definition (ffn_row in slot
    order, fmaf combine) bit for bit."""
    import torch

    from paper_2510_19470_b200 import synthetic

    H, F, E, k, G, T, stride = 128, 320, 8, 2, 2, 40, 3
    g = torch.Generator().manual_seed(31)
    dt = torch.bfloat16 if bf16 else torch.float32
    x = synthetic.dyadic((G, T, H), g, dtype=dt).float().numpy()
    wg = synthetic.dyadic((H, E), g).numpy()
    w_up, w_down = synthetic.experts(E, H, F, g, dtype=dt)
    w_up, w_down = w_up.float().numpy(), w_down.float().numpy()
    ref = oracle.moe_layer(x, wg, w_up, w_down, k, [2], [1], bf16=bf16, stride=stride)
    for gg in range(G):
        for t in range(0, T, stride):
            acc = np.zeros(H, np.float32)
            for j in range(k):
                e = ref["topk_idx"][gg, t, j]
                out = oracle.ffn_row(x[gg, t], w_up[e], w_down[e], bf16)
                acc = (np.float32(ref["topk_w"][gg, t, j]) * out.astype(np.float64) + acc).astype(np.float32)
            want = acc
            got = ref["y"][gg, t]
            if bf16:
                want = torch.from_numpy(want).to(torch.bfloat16).float().numpy()
            np.testing.assert_allclose(got, want, rtol=0, atol=0)
