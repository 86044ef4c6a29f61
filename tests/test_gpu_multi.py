"""N-GPU layer parity (NCCL dispatch / combine / expert All-Gather / SR migration).
Runs tests/mgpu_worker.py under torch.distributed.run on as many GPUs as the box has;
cases needing more GPUs than present are skipped."""
import os
import socket
import subprocess
import sys

import pytest
import torch

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
    ([2, 2, 2], [1, 2, 2], ["--E", "64", "--k", "6", "--sr"]),  # cfg4 hierarchy with migration
    # ragged: a different token count on every rank (the last rank routes one token),
    # then a second forward with the counts rotated through the same buffers
    ([2], [1], ["--ragged"]),
    ([2, 2], [1, 2], ["--ragged"]),
    ([2, 2], [2, 1], ["--ragged", "--sr"]),
    ([2, 2], [1, 1], ["--ragged", "--dtype", "f32", "--E", "16", "--k", "4"]),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("comm", ["p2p", "nccl"])
@pytest.mark.parametrize("sf,sed,extra", CASES, ids=lambda v: str(v))
def test_multi_gpu_layer(sf, sed, extra, comm):
    """comm=p2p: fused NVLink peer-memory dispatch/combine (default product path);
    comm=nccl: the NCCL grouped send/recv baseline (HEP_COMM=nccl)."""
    G = 1
    for s in sf:
        G *= s
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(HERE, "mgpu_worker.py"),
           "--sf", *map(str, sf), "--sed", *map(str, sed), *extra]
    env = dict(os.environ, HEP_COMM=comm, HEP_P2P_TIMEOUT_S="60")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
