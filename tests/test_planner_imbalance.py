"""The bench planner's load-imbalance term (CPU): per-GPU rows of a hierarchy from the
route table and the routing counts, and the choice it makes on skewed vs even routing."""
import importlib.util
import os

import pytest

from paper_2510_19470_b200 import topology as topo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)

CFG = dict(H=4096, F=14336, E=8, k=2, T=16384, dtype="bf16")
CAL = {"pre_expert_s": 1.26e-4, "expert_s_per_routed_row": 1.49e-7, "gemm_flops_per_s": 1.58e15,
       "nvlink_bytes_per_s": 4.5e11}


def test_layer_imbalance_ep_vs_allgather():
    # 2 GPUs, 4 experts each; every token of both GPUs goes to experts 0-3 (owned by GPU 0)
    counts = [[[100, 100, 100, 100, 0, 0, 0, 0], [100, 100, 100, 100, 0, 0, 0, 0]]]
    ep = topo.route_table(topo.ClusterSpec.of([2], [1]))
    ag = topo.route_table(topo.ClusterSpec.of([2], [2]))
    assert bench.layer_imbalance(counts, ep, 4) == pytest.approx(2.0)  # GPU 0 computes everything
    assert bench.layer_imbalance(counts, ag, 4) == pytest.approx(1.0)  # each GPU its own tokens


@pytest.mark.parametrize("skewed", [False, True])
def test_imbalance_plan_choice(skewed):
    G, E, rows = 4, 8, 16384 * 2
    if skewed:  # every GPU sends 70% of its rows to GPU 0's experts
        per = [int(0.35 * rows)] * 2 + [int(0.05 * rows)] * 6
    else:
        per = [rows // E] * E
    counts = [[per[:] for _ in range(G)] for _ in range(8)]
    sed, table = bench.imbalance_plan(CFG, [2, 2], G, CAL, counts)
    assert {tuple(r["sed"]) for r in table} == {(1, 1), (1, 2), (2, 1), (2, 2)}
    ref_best = min(table, key=lambda r: r["model_total_s"])["sed"]
    if skewed:
        assert sed != [1, 1]  # the term moves the choice off pure expert parallelism
    else:
        assert sed == ref_best  # even routing: the reference's own choice
