"""The multi-GPU data path on ONE GPU: every rank of the hierarchy as a virtual rank of one
process (hep_comm_init_virtual), so the driver's one-GPU box runs the fused peer-memory
step -- count exchange, dispatch stores into peers' receive areas, the down-projection's
peer-store epilogue, epoch flags, expert All-Gather pulls, SR migration and the
shared-expert chain -- against the oracle.  One subprocess per case (tests/vrank_worker.py)
under a timeout, with HEP_P2P_TIMEOUT_S so a lost flag traps with a diagnostic instead of
hanging."""
import os
import subprocess
import sys

import numpy as np

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # (sf, sed, extra args)
    ([2], [1], []),                    # pure A2A (standard EP)
    ([2], [2], []),                    # pure All-Gather
    ([2], [2], ["--sr"]),              # All-Gather of SR-migrated experts
    ([2], [1], ["--dtype", "f32", "--H", "1024", "--F", "4096", "--T", "512"]),  # cfg1/2 shape, fp32
    ([4], [2], []),
    ([2, 2], [1, 2], []),
    ([2, 2], [2, 1], ["--sr"]),
    ([2, 2], [1, 1], ["--E", "64", "--k", "6", "--H", "512", "--F", "256"]),   # fine-grained experts
    ([2, 4], [1, 4], []),              # cfg1 / cfg3 hierarchy
    ([2, 4], [1, 2], []),              # ambiguous relay (S2 tie-break)
    ([2, 4], [2, 2], []),
    ([2, 4], [1, 1], []),              # pure A2A over 8 ranks
    ([2, 4], [2, 4], []),              # pure All-Gather over 8 ranks
    ([2, 4], [1, 4], ["--dtype", "f32", "--H", "1024", "--F", "4096", "--T", "512"]),  # cfg1 itself
    ([2, 2, 2], [1, 2, 2], ["--E", "64", "--k", "6", "--sr"]),  # cfg4 hierarchy with migration
    ([2, 2, 2], [2, 1, 2], ["--E", "64", "--k", "6"]),
    # ragged: a different token count on every rank, rotated, then rank 0 empty
    ([2], [1], ["--ragged"]),
    ([2, 2], [1, 2], ["--ragged"]),
    ([2, 2], [2, 1], ["--ragged", "--sr"]),
    ([2, 4], [1, 2], ["--ragged"]),
    ([2, 2], [1, 1], ["--ragged", "--dtype", "f32", "--E", "16", "--k", "4"]),
    # the residual form y = x + MoE(x), fused into the combine (bf16 local combine, fp32 p2p combine)
    ([2, 2], [1, 2], ["--residual"]),
    ([2], [1], ["--residual", "--dtype", "f32", "--H", "1024", "--F", "4096", "--T", "512"]),
    # weights rewritten between steps while peers pull them (dense and SR All-Gather)
    ([2, 4], [1, 4], ["--update"]),
    ([2, 2, 2], [1, 2, 2], ["--E", "64", "--k", "6", "--sr", "--update"]),
    # the optimizer step fused with the migration encode, then a step on the new experts
    ([2, 2], [2, 1], ["--sr", "--sgd"]),
    ([2, 2, 2], [1, 2, 2], ["--E", "64", "--k", "6", "--sr", "--sgd"]),
    # a corrupted migrated expert is rejected (RuntimeFailure), not consumed silently
    ([2, 2], [1, 2], ["--sr", "--corrupt"]),
    # ranks that disagree on the layer shape are rejected before any peer store
    ([2], [1], ["--mismatch"]),
]


@pytest.mark.parametrize("sf,sed,extra", CASES, ids=lambda v: str(v))
def test_virtual_ranks_layer(sf, sed, extra):
    cmd = [sys.executable, os.path.join(HERE, "vrank_worker.py"), "--sf", *map(str, sf), "--sed", *map(str, sed),
           *extra]
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", HEP_P2P_TIMEOUT_S="60")
    env.pop("HEP_COMM", None)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=420, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    if "--mismatch" in extra:
        assert "mismatch rejected" in r.stdout, r.stdout[-2000:]
    else:
        assert r.stdout.count(" ok ") >= 2, r.stdout[-2000:]


# The step's opt-in schedules must compute the same thing: one GEMM launch per projection
# over every group (HEP_MERGE_GEMMS=1), own + received merged (=2), a capped grid-stride
# remote dispatch (HEP_DISPATCH_CTAS: several rows per warp), the All-Gather stream at
# top priority (HEP_AG_PRIORITY=1).
SCHEDULE_CASES = [
    ({"HEP_MERGE_GEMMS": "1"}, [2, 2, 2], [1, 2, 2], ["--E", "64", "--k", "6", "--sr"]),
    ({"HEP_MERGE_GEMMS": "1"}, [2, 4], [1, 2], ["--ragged"]),
    ({"HEP_MERGE_GEMMS": "2"}, [2, 2], [2, 1], ["--sr", "--ragged"]),
    ({"HEP_MERGE_GEMMS": "2"}, [2, 4], [1, 4], []),
    ({"HEP_DISPATCH_CTAS": "3"}, [2, 4], [1, 1], ["--ragged"]),
    ({"HEP_DISPATCH_CTAS": "16", "HEP_AG_PRIORITY": "1"}, [2, 2, 2], [1, 2, 2], ["--E", "64", "--k", "6", "--sr"]),
]


@pytest.mark.parametrize("envs,sf,sed,extra", SCHEDULE_CASES, ids=lambda v: str(v))
def test_virtual_ranks_schedules(envs, sf, sed, extra):
    cmd = [sys.executable, os.path.join(HERE, "vrank_worker.py"), "--sf", *map(str, sf), "--sed", *map(str, sed),
           *extra]
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", HEP_P2P_TIMEOUT_S="60", **envs)
    env.pop("HEP_COMM", None)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=420, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    assert r.stdout.count(" ok ") >= 2, r.stdout[-2000:]


FUSED_CASES = [
    ([2], [2], ["--sr"]),
    ([2, 2, 2], [1, 2, 2], ["--E", "64", "--k", "6", "--sr", "--update"]),
    ([2, 2], [2, 1], ["--ragged", "--sr"]),
    ([2, 2], [2, 1], ["--sr", "--sgd"]),
    ([2, 2], [1, 2], ["--sr", "--corrupt"]),
]


@pytest.mark.parametrize("sf,sed,extra", FUSED_CASES, ids=lambda v: str(v))
def test_virtual_ranks_layer_fused_decode(sf, sed, extra):
    """The SR cases with the decode fused into the expert GEMM (HEP_SR_FUSED=1)."""
    cmd = [sys.executable, os.path.join(HERE, "vrank_worker.py"), "--sf", *map(str, sf), "--sed", *map(str, sed),
           *extra]
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", HEP_P2P_TIMEOUT_S="60", HEP_SR_FUSED="1")
    env.pop("HEP_COMM", None)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=420, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    assert r.stdout.count(" ok ") >= 2, r.stdout[-2000:]


@pytest.mark.parametrize("sf,sed,extra", [
    ([2, 2], [2, 1], []),
    ([2, 2, 2], [1, 2, 2], ["--E", "64", "--k", "6"]),
    ([2], [2], ["--H", "2048", "--F", "1408", "--E", "8", "--T", "512"]),
], ids=lambda v: str(v))
@pytest.mark.parametrize("pair", ["1", "0"], ids=["cta_pair", "single_cta"])
def test_fused_decode_gemm_inputs_bit_identical(sf, sed, extra, pair, tmp_path):
    """SR decode fused into the GEMM's B-operand load vs the dense decode into compute
    copies: with the same GEMM (CTA pair, or 1-CTA) for both, every rank's output is
    bit-identical, so the patched B tiles equal the dense-decoded expert exactly."""
    outs = []
    for fused in ("1", "0"):
        dump = str(tmp_path / f"y_{fused}.npy")
        cmd = [sys.executable, os.path.join(HERE, "vrank_worker.py"), "--sf", *map(str, sf), "--sed", *map(str, sed),
               "--sr", "--dump", dump, *extra]
        env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", HEP_P2P_TIMEOUT_S="60", HEP_SR_FUSED=fused,
                   HEP_GEMM_2CTA=pair)
        env.pop("HEP_COMM", None)
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=420, env=env)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
        outs.append(np.load(dump))
    assert outs[0].shape == outs[1].shape
    assert np.array_equal(outs[0], outs[1]), int((outs[0] != outs[1]).sum())
