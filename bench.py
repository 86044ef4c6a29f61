"""MoE-layer tokens/s on B200 (BASELINE.json metric), one process per GPU.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config cfg3]

Workload (default cfg3, BASELINE.json configs[2]): one Mixtral-8x7B-shaped MoE layer,
bf16, H=4096, F=14336, E=8, top-2, 16,384 tokens per GPU (weak scaling), synthetic
data.  configs[1] (cfg2, the fp32 S_ED sweep at 512 tokens/GPU) is a parity case, not a
bench line.  A step = one full layer pass through the public API:
expert All-Gather (N > 1) + gate + permute + dispatch + expert FFN + combine.

value : tokens/s of all ranks, inputs resident in HBM, device-timed (CUDA events on
        the launching stream), max over ranks.
e2e   : same metric through hep_layer_forward_host (pinned host x -> H2D -> step ->
        D2H of y) -- the reference-facing call with host buffers.
roofline : the expert grouped GEMM (K8), FLOPs / its launch time measured live with
        CUDA events on the launching stream IN the timed `value` pass (phase events at
        every kernel boundary of every step), vs the measured sustained bf16 peak of
        MEASURED_PEAKS.json (burst fraction beside it); `kernels` gives the same pass's
        gate / permute / combine times as fractions of measured HBM bandwidth.
planner : at N > 1 the S_ED of cfg3/cfg5 comes from the reference's solver fed numbers
        measured in this run (calibration: pre-expert time and expert-GEMM rate of a
        one-GPU layer of the same shape, NVLink bytes/s of an NCCL all-gather); the
        plan.json / freq.json / topo.csv reports are written in the reference's formats.
cpu_baseline : the CPU oracle (oracle/moe_oracle.c, OpenMP) on a bounded token sample.
--impl reference : times that same CPU implementation as the reference arm (the
        reference has no GPU path and no gate/FFN/combine of its own),
        with inputs generated on the CPU: that arm never loads libhep.so or touches a GPU.
"""
from __future__ import annotations

import argparse
import gc
import json
import os

# separate hardware queues for the step's streams (see paper_2510_19470_b200/__init__.py);
# set before torch creates the CUDA context
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg3": dict(workload="cfg3: Mixtral-8x7B-shaped MoE layer (8 experts top-2, d=4096, FFN 14336), bf16",
                 H=4096, F=14336, E=8, k=2, T=16384, dtype="bf16", layers=1, sr=False,
                 # SF per N; S_ED = the reference planner's pick on measured B200 numbers
                 # (cfg3: "S_ED pinned [1,4] plus the solver's pick"; the pinned [1,4] at N=8
                 # is `--sed 1,4`).
                 topo={1: ([1], [1]), 2: ([2], None), 4: ([2, 2], None), 8: ([2, 4], None)}),
    "cfg4": dict(workload="cfg4: DeepSeek-style fine-grained MoE layer (64 experts top-6, d=2048, FFN 1408), bf16, "
                          "SR-migrated experts (CR=50)",
                 H=2048, F=1408, E=64, k=6, T=16384, dtype="bf16", layers=1, sr=True,
                 topo={1: ([1], [1]), 2: ([2], [2]), 4: ([2, 2], [1, 2]), 8: ([2, 2, 2], [1, 2, 2])}),
    "cfg5": dict(workload="cfg5: 8-layer stack of Mixtral-shaped MoE layers, bf16, S_ED from perf::solve_optimal_p "
                          "on measured B200 numbers",
                 H=4096, F=14336, E=8, k=2, T=16384, dtype="bf16", layers=8, sr=False,
                 topo={1: ([1], [1]), 2: ([2], None), 4: ([2, 2], None), 8: ([2, 4], None)}),
    "cfg1": dict(workload="cfg1/cfg2 shape: 8 experts top-2, d=1024, FFN 4096, 512 tokens/GPU, fp32",
                 H=1024, F=4096, E=8, k=2, T=512, dtype="f32", layers=1, sr=False,
                 topo={1: ([1], [1]), 2: ([2], [1]), 4: ([2, 2], [1, 1]), 8: ([2, 4], [1, 4])}),
}

def calibrate(cfg, dev, dtype, world, MoELayer):
    """Planner inputs measured on this GPU: a one-GPU layer of the
    config's shape (all E experts local) times gate + scans + permute (the pre-expert
    stream) and the expert GEMM pair (C = 4HF FLOPs per routed row / GEMM time); an NCCL
    all-gather of 64 MB per rank gives the NVLink bytes/s each GPU receives (B)."""
    import torch
    import torch.distributed as dist

    H, F, E, k, T = cfg["H"], cfg["F"], cfg["E"], cfg["k"], cfg["T"]
    x, wg = make_inputs(cfg, 0, dev, dtype)
    layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=dtype)
    layer.set_gate(wg)
    for e in range(E):
        u, d = expert_weights(cfg, e, dev, dtype)
        layer.set_expert(e, u, d)
        del u, d
    y = torch.empty_like(x)
    for _ in range(3):
        layer.forward(x, out=y)
    layer.set_profiling(True)
    layer.timings()
    for _ in range(5):
        layer.forward(x, out=y)
    ph = layer.timings()
    layer.close()
    del layer, y
    torch.cuda.empty_cache()
    pre = (ph.get("gate", 0.0) + ph.get("scan", 0.0) + ph.get("permute", 0.0)) / 1e3
    gemm = sum(v for n, v in ph.items() if n.startswith("gemm_")) / 1e3
    rows = T * k
    out = {"pre_expert_s": pre, "expert_s_per_routed_row": gemm / rows, "gemm_flops_per_s": 4.0 * H * F * rows / gemm,
           "source": "measured in this run: one-GPU layer of this shape, 5 profiled forwards"}
    if world > 1:
        n = 64 << 20
        buf = torch.empty(n, dtype=torch.uint8, device=dev)
        gat = torch.empty(world * n, dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(gat, buf)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dist.all_gather_into_tensor(gat, buf)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 5 / 1e3], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["nvlink_bytes_per_s"] = (world - 1) * n / float(t.item())
        del buf, gat
    return out


def planned_sed(cfg, sf, world, cal, report_dir):
    """cfg3/cfg5 at N > 1: the reference solver (perfmodel.cpp:200-217, via
    hep_plan_reports) on this run's measured numbers, the innermost-first split
    (plan.cpp:41-58), and the reference's plan.json / freq.json / topo.csv."""
    from paper_2510_19470_b200 import topology as topo
    n = cfg["E"] // world
    rows = cfg["T"] * cfg["k"]
    b = 2 if cfg["dtype"] == "bf16" else 4
    p, sed, lat = topo.plan_reports(
        topo.ClusterSpec.of(sf, [1] * len(sf), bandwidth=cal["nvlink_bytes_per_s"]),
        data_size_D=float(rows * cfg["H"] * b), expert_size_PE=float(n * 2 * cfg["H"] * cfg["F"] * b),
        experts_per_gpu_n=n, attn_latency=cal["pre_expert_s"],
        expert_latency=cal["expert_s_per_routed_row"] * rows / n, throughput_C=cal["gemm_flops_per_s"],
        bandwidth_B=cal["nvlink_bytes_per_s"], out_dir=report_dir)
    return sed, p, lat


def imbalance_plan(cfg, sf, world, cal, counts):
    """The reference's model (hep_plan_reports with each S_ED pinned) plus a load-imbalance
    term: total + comp * (imbalance - 1), where imbalance is the busiest GPU's GEMM rows
    over the mean under that hierarchy, from this run's routing (counts[l][s][e] = rows
    of layer l that source GPU s routes to expert e; route_table gives the computing GPU
    of every (source, owner) pair), averaged over the layers.  The reference's model
    assumes evenly activated experts and its compute term does not depend
    on S_ED, so on skewed routing it keeps choosing pure expert parallelism
    (profiles/r2_cfg5_sweep/).  Returns (chosen S_ED, candidate table)."""
    import itertools
    from paper_2510_19470_b200 import topology as topo
    n = cfg["E"] // world
    rows = cfg["T"] * cfg["k"]
    b = 2 if cfg["dtype"] == "bf16" else 4
    divs = [[d for d in range(1, f + 1) if f % d == 0] for f in sf]
    table = []
    for sed in itertools.product(*divs):
        sed = list(sed)
        p, got, lat = topo.plan_reports(
            topo.ClusterSpec.of(sf, [1] * len(sf), bandwidth=cal["nvlink_bytes_per_s"]),
            data_size_D=float(rows * cfg["H"] * b), expert_size_PE=float(n * 2 * cfg["H"] * cfg["F"] * b),
            experts_per_gpu_n=n, attn_latency=cal["pre_expert_s"],
            expert_latency=cal["expert_s_per_routed_row"] * rows / n, throughput_C=cal["gemm_flops_per_s"],
            bandwidth_B=cal["nvlink_bytes_per_s"], pinned_sed=sed)
        imb = layer_imbalance(counts, topo.route_table(topo.ClusterSpec.of(sf, sed)), n)
        table.append({"sed": sed, "p": p, "model_total_s": lat["total"], "imbalance": imb,
                      "model_with_imbalance_s": lat["total"] + lat["comp"] * (imb - 1.0)})
    best = min(table, key=lambda r: r["model_with_imbalance_s"])
    return best["sed"], table


def layer_imbalance(counts, route, n):
    """Mean over layers of max / mean GPU rows, counts[l][s][e] routed under route[s][owner]."""
    G = len(route)
    vals = []
    for per_layer in counts:
        load = [0] * G
        for s_ in range(G):
            for e, c in enumerate(per_layer[s_]):
                load[int(route[s_][e // n])] += int(c)
        mean = sum(load) / G
        vals.append(max(load) / mean if mean > 0 else 1.0)
    return sum(vals) / len(vals)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--cpu-stride", type=int, default=64)
    p.add_argument("--sed", default="", help="override S_ED per level, e.g. 1,4")
    p.add_argument("--planner", default="imbalance", choices=["imbalance", "reference"],
                   help="cfg3/cfg5 at N>1: the reference's model plus this run's measured routing imbalance "
                        "(default), or the reference's model alone")
    p.add_argument("--report-dir", default="", help="where the planner reports go (default gpurun_out/plan_reports)")
    return p.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: an NVML polling
    thread every 25 ms plus one sample as the region opens (in __enter__) and one as it
    closes (in __exit__), so even a few-ms region of a small config is covered;
    nvidia-smi -lms 50 if NVML is absent.  (Polling every 2 ms stalled cfg1's launch-bound
    4-GPU step by up to 5x.)"""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc, self.nvml = index, [], None, None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _sample(self):
        p = self.nvml
        sm = p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM)
        bits = p.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.rows.append((float(sm), float(self.max_sm), [n for n, b in self.REASONS if bits & b]))

    def _poll(self):
        while not self.stop.wait(0.025):
            try:
                self._sample()
            except Exception:
                return

    def _read(self):
        names = [n for n, _ in self.REASONS]
        for line in self.proc.stdout:
            r = [c.strip() for c in line.split(",")]
            if len(r) >= 8 and r[1].replace(".", "").isdigit():
                self.rows.append((float(r[1]), float(r[2]), [names[i] for i in range(4) if r[4 + i] == "Active"]))

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            try:
                self._sample()  # one sample at the end of the region
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows]
        reasons = sorted({n for r in self.rows for n in r[2]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


def make_inputs(cfg, rank, device, dtype):
    import torch
    from paper_2510_19470_b200 import synthetic

    g = torch.Generator(device=device).manual_seed(1000 + rank)
    x = synthetic.dyadic((cfg["T"], cfg["H"]), g, device=device, dtype=dtype)
    gw = torch.Generator(device=device).manual_seed(7)
    wg = synthetic.dyadic((cfg["H"], cfg["E"]), gw, device=device)
    return x, wg


def expert_weights(cfg, e, device, dtype):
    """Expert e of the demo population (shared base from seed 11, per-expert noise)."""
    import torch
    from paper_2510_19470_b200.synthetic import expert_scale

    H, F = cfg["H"], cfg["F"]
    s = expert_scale(H)
    gb = torch.Generator(device=device).manual_seed(11)
    ge = torch.Generator(device=device).manual_seed(100 + e)

    def mat(shape):
        base = (0.05 + 0.95 * torch.rand(shape, generator=gb, device=device)) * \
            (torch.randint(0, 2, shape, generator=gb, device=device) * 2 - 1)
        noise = (torch.rand(shape, generator=ge, device=device) * 2 - 1) * 0.05
        return ((base + noise) * s).to(dtype)

    return mat((H, F)), mat((F, H))


def cpu_oracle_inputs(cfg, x=None, wg=None):
    """The same synthetic workload as the GPU arm, as fp32 host arrays for the oracle."""
    import numpy as np
    import torch

    H, F, E = cfg["H"], cfg["F"], cfg["E"]
    dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    if x is None:
        x, wg = make_inputs(cfg, 0, dev, dt)
    ups = np.empty((E, H, F), np.float32)
    downs = np.empty((E, F, H), np.float32)
    for e in range(E):
        u, d = expert_weights(cfg, e, dev, dt)
        ups[e] = u.float().cpu().numpy()
        downs[e] = d.float().cpu().numpy()
    return x.float().cpu().numpy()[None], wg.float().cpu().numpy(), ups, downs


def cpu_oracle_time(cfg, inputs, stride):
    """Times the CPU oracle (all host threads) on every `stride`-th token of one GPU's
    workload; routing covers every token.  Returns (tokens/s, seconds, sampled, threads)."""
    import oracle

    xs, wgs, ups, downs = inputs
    t0 = time.perf_counter()
    oracle.moe_layer(xs, wgs, ups, downs, cfg["k"], [1], [1], bf16=cfg["dtype"] == "bf16", stride=stride)
    secs = time.perf_counter() - t0
    sampled = (cfg["T"] + stride - 1) // stride
    # a step of an L-layer stack is L layer passes (cfg5); the sample times one of them
    return sampled / (secs * cfg.get("layers", 1)), secs, sampled, oracle.num_threads()


def cpu_inputs(cfg):
    """The same synthetic workload, generated on the CPU for the reference arm (which must
    not load libhep.so or touch a GPU): dyadic tokens and gate, the reference demo expert
    population (cli_app.cpp:89-118) at the config's shape and dtype.  Distribution and
    shapes equal the GPU arm's; the CPU oracle's cost does not depend on the draw."""
    import numpy as np
    import torch

    H, F, E, T = cfg["H"], cfg["F"], cfg["E"], cfg["T"]
    dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    g = torch.Generator().manual_seed(1000)
    x = (torch.randint(-8, 9, (T, H), generator=g).float() / 16.0)
    wg = (torch.randint(-8, 9, (H, E), generator=g).float() / 16.0)
    scale = 2.0 ** -5 if H <= 1024 else 2.0 ** -6
    ups = np.empty((E, H, F), np.float32)
    downs = np.empty((E, F, H), np.float32)
    gb = torch.Generator().manual_seed(11)
    base_u = (0.05 + 0.95 * torch.rand((H, F), generator=gb)) * (torch.randint(0, 2, (H, F), generator=gb) * 2 - 1)
    base_d = (0.05 + 0.95 * torch.rand((F, H), generator=gb)) * (torch.randint(0, 2, (F, H), generator=gb) * 2 - 1)
    for e in range(E):
        ge = torch.Generator().manual_seed(100 + e)
        ups[e] = ((base_u + (torch.rand((H, F), generator=ge) * 2 - 1) * 0.05) * scale).to(dt).float().numpy()
        downs[e] = ((base_d + (torch.rand((F, H), generator=ge) * 2 - 1) * 0.05) * scale).to(dt).float().numpy()
    return x.to(dt).float().numpy()[None], wg.numpy(), ups, downs


def run_reference(args, cfg):
    """Reference arm: the CPU implementation of the path, rank 0 only, CPU inputs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    inputs = cpu_inputs(cfg)
    vals = []
    for i in range(args.warmup + args.steps):
        tps, secs, sampled, cores = cpu_oracle_time(cfg, inputs, args.cpu_stride)
        if i >= args.warmup:
            vals.append(tps)
    v = statistics.median(vals)
    sample = f"every {args.cpu_stride}th of {cfg['T']} tokens ({sampled} tokens) through the full layer per step"
    line = {"impl": "reference", "metric": "MoE-layer tokens/s", "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sampled / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic (generated on the CPU)", "config": {"workload": cfg["workload"], "tokens_per_gpu": cfg["T"]},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bind_to_gpu_numa(device_index):
    """Pin this rank's host threads to the CPUs NVML reports as local to its GPU, so the
    pinned host buffers of the e2e leg are first-touched on the GPU's NUMA node (the
    H2D/D2H traffic of all ranks then stays off the socket interconnect)."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        bus = torch.cuda.get_device_properties(device_index).pci_bus_id
        dom = torch.cuda.get_device_properties(device_index).pci_domain_id
        dev = torch.cuda.get_device_properties(device_index).pci_device_id
        h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{dom:08x}:{bus:02x}:{dev:02x}.0")
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
        return sorted(cpus)
    except Exception:
        return None


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    from paper_2510_19470_b200 import synthetic
    from paper_2510_19470_b200.moe import Communicator, MoELayer, gather_all

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    numa_cpus = bind_to_gpu_numa(local) if world > 1 else None
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = Communicator.from_torch()
    sf, sed = cfg["topo"][world]
    dtype = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    p_plan = planner = None
    if args.sed:
        sed = [int(v) for v in args.sed.split(",")]
    elif sed is None:
        cal = calibrate(cfg, dev, dtype, world, MoELayer)
        report_dir = args.report_dir or os.path.join(ROOT, "gpurun_out", "plan_reports", f"{args.config}_n{world}")
        sed, p_plan, lat = planned_sed(cfg, sf, world, cal, report_dir if rank == 0 else None)
        planner = {"measured_inputs": cal, "p": p_plan, "sed": sed, "modelled_latency_s": lat,
                   "reports": os.path.relpath(report_dir, ROOT) + "/{plan.json,freq.json,topo.csv}"}
    sed_source = "override" if args.sed else ("planner" if p_plan is not None else "pinned")
    H, F, E, k, T = cfg["H"], cfg["F"], cfg["E"], cfg["k"], cfg["T"]
    use_sr = cfg["sr"] and world > 1
    srcfg = None
    if use_sr:
        from paper_2510_19470_b200.sr import CompressionConfig
        srcfg = CompressionConfig(ratio_CR=50.0)

    x, wg = make_inputs(cfg, rank, dev, dtype)

    def build_stack(sed):
        layers = []
        for li in range(cfg["layers"]):
            layers.append(build_layer(li, sed))
        torch.cuda.synchronize()
        return layers

    def build_layer(li, sed):
        layer = MoELayer(hidden=H, ffn=F, experts=E, top_k=k, max_tokens=T, dtype=dtype, sf=sf, sed=sed, rank=rank,
                         comm=comm, sr=srcfg)
        if li == 0:
            layer.set_gate(wg)
        else:
            # every layer of a stack has its own gate (as the architecture does); one gate
            # shared by all 8 layers collapses the routing of the chained activations onto a
            # few experts
            gl = torch.Generator(device=dev).manual_seed(7 + li)
            layer.set_gate(synthetic.dyadic((H, E), gl, device=dev))
        if use_sr:
            # shared expert = mean of the population (the reference's init_shared); the demo
            # population shares one base, so every rank computes the same mean locally.
            from paper_2510_19470_b200 import sr as srmod
            acc = None
            for e in range(E):
                u, d = expert_weights(cfg, e, dev, dtype)
                flat = torch.cat([u.float().reshape(-1), d.float().reshape(-1)])
                acc = flat.double() if acc is None else acc + flat.double()
            layer.set_shared((acc / E).float().contiguous())
            del acc
        for e in layer.owned_experts():
            u, d = expert_weights(cfg, e + 1000 * li, dev, dtype)
            layer.set_expert(e, u, d)
            del u, d
        return layer

    layers = build_stack(sed)
    acts = [x] + [torch.empty_like(x) for _ in range(cfg["layers"])]
    if p_plan is not None and args.planner == "imbalance":
        # this run's routing: one pass of the stack (routing does not depend on S_ED), the
        # rows every source GPU sends to every expert per layer, gathered from all ranks
        if world > 1:
            gather_all(layers)
        for li, layer in enumerate(layers):
            layer.forward(acts[li], out=acts[li + 1], residual=len(layers) > 1)
        torch.cuda.synchronize()
        mine = torch.stack([layer.debug(T)["key_counts"].to(dev).long().view(world, E).sum(0) for layer in layers])
        allc = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allc, mine)
        counts = torch.stack(allc, 1).cpu().tolist()  # [layer][source][expert]
        choice, table = imbalance_plan(cfg, sf, world, cal, counts)
        planner.update({"reference_sed": sed, "sed": choice, "mode": "reference model + measured routing imbalance",
                        "candidates": table})
        p_plan = next(r["p"] for r in table if r["sed"] == choice)
        planner["p"] = p_plan
        if choice != sed:
            for layer in layers:
                layer.close()
            del layers
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            sed = choice
            layers = build_stack(sed)

    def step():
        if world > 1:
            # every layer's expert All-Gather queued at t=0 (simcore.cpp:155-174); the
            # pulls run on the copy engines under the layers' compute
            gather_all(layers)
        for li, layer in enumerate(layers):
            # a stack applies each layer on the residual stream, y = x + MoE(x) (the add is
            # fused into the combine): chained raw MoE outputs would route ever more unevenly
            layer.forward(acts[li], out=acts[li + 1], residual=len(layers) > 1)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------------------------------------------------------- device-timed region
    # Bring the SM clocks up from idle first (200 ms of torch bf16 matmuls, none of our
    # kernels): the W warm-up steps of a small config last ~1 ms, far shorter than the
    # clock ramp, and a cfg1 value taken straight after setup read 40% low.
    ramp = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    r0 = torch.cuda.Event(enable_timing=True)
    r1 = torch.cuda.Event(enable_timing=True)
    r0.record()
    while True:
        for _ in range(20):
            ramp2 = ramp @ ramp
        r1.record()
        r1.synchronize()
        if r0.elapsed_time(r1) >= 200.0:
            break
    del ramp, ramp2
    # The timed pass carries CUDA events around every expert-GEMM launch of every step (on
    # the launching stream): the GEMM time the roofline divides by comes from the same K
    # steps as `value`.  Events at every phase boundary cost the launch-bound small configs
    # up to 2x (cfg1 at 4 GPUs), so the per-phase times and the HBM kernels' fractions come
    # from a second, fully instrumented pass of the same K steps right after.
    for layer in layers:
        layer.set_profiling(1)
    for _ in range(args.warmup):
        step()
    # The clock sampler starts before the last barrier: its NVML initialisation takes a
    # different time on every rank, and a rank that opens the timed region early counts
    # its peers' lateness in its first step (40-100 ms outliers at N=4 before this).
    clocks = ClockSampler(local).__enter__()
    gc.disable()  # no collector pauses inside the timed passes (launch-bound configs feel them)
    for layer in layers:
        layer.timings()  # drop the warm-up marks
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # an event at every step boundary too (K records, no syncs): the per-step spread shows
    # a host stall inside the timed region, which the total alone cannot
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps - 1)]
    barrier()
    t0.record(stream)
    for i in range(args.steps):
        step()
        if i < args.steps - 1:
            marks[i].record(stream)
    t1.record(stream)
    barrier()
    ms = t0.elapsed_time(t1)
    bounds = [t0] + marks + [t1]
    per_step = sorted(bounds[i].elapsed_time(bounds[i + 1]) for i in range(args.steps))
    step_spread = {"min": per_step[0], "median": per_step[len(per_step) // 2], "max": per_step[-1],
                   "source": "CUDA events at every step boundary of the timed pass (rank 0)"}
    gemm_phases = {}  # mean ms per step, summed over the layers of the stack
    for layer in layers:
        for kname, v in layer.timings().items():
            gemm_phases[kname] = gemm_phases.get(kname, 0.0) + v
        layer.set_profiling(2)
    for _ in range(args.steps):
        step()
    barrier()
    phases = {}
    for layer in layers:
        for kname, v in layer.timings().items():
            phases[kname] = phases.get(kname, 0.0) + v
        layer.set_profiling(0)
    launches = sum(layer.launch_count() for layer in layers) * args.steps
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * T * args.steps / (ms_max / 1000.0)

    # Rows this GPU's expert GEMMs processed in one step (local + received), all layers.
    # key_counts[d*E + e] = this GPU's rows for expert e computed on GPU d; summed over the
    # sources, the slice d = rank is every row this GPU's GEMMs ran (local, received and
    # rows for gathered experts)
    rows = 0
    rows_per_gpu = [0] * world  # every GPU's GEMM rows per step: the load balance of the routing
    layer_imbalance = []        # per layer: max over GPUs of its GEMM rows / the mean
    for layer in layers:
        kc = layer.debug(T)["key_counts"].to(dev).long()
        if world > 1:
            dist.all_reduce(kc)
        rows += int(kc[rank * E:(rank + 1) * E].sum().item())
        per = [int(kc[d * E:(d + 1) * E].sum().item()) for d in range(world)]
        for d in range(world):
            rows_per_gpu[d] += per[d]
        layer_imbalance.append(max(per) * world / max(1, sum(per)))
    gemm_ms = sum(v for kname, v in gemm_phases.items() if kname.startswith("gemm_"))
    step_ms_local = ms / args.steps
    assert gemm_ms <= step_ms_local * 1.001, f"GEMM time {gemm_ms:.4f} ms exceeds the step {step_ms_local:.4f} ms"
    pk = peaks()
    flops = 4.0 * H * F * rows
    achieved = flops / (gemm_ms / 1000.0) / 1e12 if gemm_ms > 0 else None
    peak = pk.get("bf16_tflops_sustained", 1400.0)
    peak_burst = pk.get("bf16_tflops", 1590.0)
    peak_source = ("MEASURED_PEAKS.json bf16_tflops_sustained (the GEMM is timed inside a back-to-back step loop "
                   "under sw_power_cap, the regime of the sustained figure; see clocks)")
    gemm_kernel = "grouped expert GEMM (up+down, tcgen05 kind::f16)"
    if cfg["dtype"] == "f32":
        # fp32 layers run 3xTF32 on the tensor cores: TF32 is half the bf16 rate and every
        # fp32 product costs three TF32 MMAs, so the fp32-equivalent ceiling is bf16 / 6
        peak = peak / 6.0
        peak_burst = peak_burst / 6.0
        peak_source = "derived: MEASURED_PEAKS.json bf16_tflops_sustained / 2 (tf32 rate) / 3 (3xTF32 MMAs per product)"
        gemm_kernel = "grouped expert GEMM (up+down, tcgen05 kind::tf32, 3xTF32)"
    # HBM-bound kernels of the same pass (SURVEY §8(d) algorithmic bytes, b = element bytes)
    b = 2 if dtype == torch.bfloat16 else 4
    L = cfg["layers"]
    hbm = pk.get("hbm_gbs", 6650.0)
    algo = {"gate": L * (T * H * b + E * H * b + T * k * 16),
            "permute": L * (T * H * b + T * k * H * b + T * k * 4),
            "combine": L * (T * k * H * b + T * k * 8 + T * H * b)}
    kernels = {}
    for kname, nbytes in algo.items():
        if phases.get(kname):
            gbs = nbytes / (phases[kname] / 1e3) / 1e9
            kernels[kname] = {"ms_per_step": phases[kname], "algorithmic_bytes": nbytes, "achieved_gbs": gbs,
                              "hbm_frac": gbs / hbm}
    for kname in ("gemm_up", "gemm_down"):
        # every launch of that projection (own, received and gathered groups at N > 1)
        t_ms = sum(v for n_, v in gemm_phases.items() if n_.startswith(kname))
        if t_ms:
            f = flops / 2.0  # up and down are 2HF FLOPs per row each
            kernels[kname] = {"ms_per_step": t_ms, "tflops": f / (t_ms / 1e3) / 1e12,
                              "frac_sustained": f / (t_ms / 1e3) / 1e12 / peak,
                              "frac_burst": f / (t_ms / 1e3) / 1e12 / peak_burst}
    kernels["hbm_peak_gbs"] = hbm
    kernels["source"] = ("gemm_*: CUDA events around the GEMM launches in the timed pass; gate/permute/combine: events "
                         "at every phase boundary in a second pass of the same K steps (launching stream)")
    # DRAM bytes of one up+down GEMM pair from an ncu capture of the same N=1 workload
    # (profiles/ncu_summary.json); the N>1 step splits the GEMM into more launches
    traffic = None
    if world == 1:
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
            traffic = prof.get(args.config, {}).get("gemm_dram_bytes_per_launch")
        except Exception:
            pass

    # ---------------------------------------------------------------- e2e through host buffers
    xh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()

    def e2e_step():
        if len(layers) == 1:
            if world > 1:
                layers[0].gather_experts()
            layers[0].forward_host(xh, yh)
        else:
            acts[0].copy_(xh, non_blocking=True)
            step()
            yh.copy_(acts[-1], non_blocking=True)

    def e2e_fence():
        if len(layers) == 1:
            layers[0].host_fence()

    for _ in range(2):
        e2e_step()
    e2e_fence()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e2e_fence()
    e1.record(stream)
    barrier()
    clocks.__exit__()
    gc.enable()
    e_ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e = world * T * args.steps / (float(e_ms.item()) / 1000.0)
    row_bytes = H * (2 if dtype == torch.bfloat16 else 4)
    layer = layers[0]

    comm_stats = None
    if world > 1:
        # A2A + AG bus bandwidth per GPU (BASELINE metric), against the measured NVLink
        # peer-copy bandwidth of B200_PROFILING.md (770 GB/s per direction).
        cb = layers[0].comm_bench(x, iters=10)
        if cb["ag_bus_gbs"] is None:
            # this plan has no All-Gather (the planner picked p=1); measure the expert
            # All-Gather the hybrid plan would run (NCCL, one GPU's expert payload)
            n = len(layers[0].owned_experts())
            payload = torch.empty(n * 2 * H * F, dtype=dtype, device=dev)
            gathered = torch.empty(world * payload.numel(), dtype=dtype, device=dev)
            dist.all_gather_into_tensor(gathered, payload)
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(5):
                dist.all_gather_into_tensor(gathered, payload)
            a1.record(stream)
            torch.cuda.synchronize()
            ag_ms = a0.elapsed_time(a1) / 5
            cb["ag_ms"], cb["ag_bytes"] = ag_ms, (world - 1) * payload.numel() * payload.element_size()
            cb["ag_bus_gbs"] = cb["ag_bytes"] / (ag_ms * 1e6)
            cb["ag_source"] = "nccl all_gather of one GPU's expert payload (torch.distributed)"
            del payload, gathered
        stats = torch.tensor([cb["a2a_bus_gbs"] or 0.0, cb["ag_bus_gbs"] or 0.0, cb.get("ag_pull_bus_gbs") or 0.0],
                             device=dev, dtype=torch.float64)
        dist.all_reduce(stats, op=dist.ReduceOp.MIN)
        # The reference's per-level stripe-model bytes of this plan (traffic_report,
        # topology.cpp:249-281) beside the physical bytes this GPU moved (SURVEY §7 hard
        # part 2: the two differ for multi-level clusters)
        from paper_2510_19470_b200 import topology as topo
        n_e = E // world
        stripe = topo.traffic_report(topo.ClusterSpec.of(sf, sed), data_size_D=float(T * k * H * b),
                                     expert_size_PE=float(n_e * 2 * H * F * b))
        comm_stats = dict(cb, a2a_bus_gbs_min_over_ranks=float(stats[0]), ag_bus_gbs_min_over_ranks=float(stats[1]),
                          nvlink_peak_gbs=770.0, peak_source="B200_PROFILING.md measured peer copy per direction",
                          a2a_frac=float(stats[0]) / 770.0, ag_frac=float(stats[1]) / 770.0,
                          ag_pull_bus_gbs_min_over_ranks=float(stats[2]), ag_pull_frac=float(stats[2]) / 770.0,
                          physical_bytes_per_gpu={"a2a_dispatch_sent": cb["a2a_bytes"], "ag_received": cb["ag_bytes"]},
                          stripe_model_bytes_cluster={"per_level": stripe, "unit": "bytes per layer pass, "
                                                      "all GPUs (traffic_report, topology.cpp:249-281)"})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        tps, secs, sampled, cores = cpu_oracle_time(cfg, cpu_oracle_inputs(cfg, x, wg), args.cpu_stride)
        cpu = {"value": tps, "unit": "tokens/s", "cores": cores, "kind": "port",
               "sample": f"every {args.cpu_stride}th of {T} tokens ({sampled} tokens) through the full layer "
                         f"(routing of all {T} tokens included), {secs:.1f} s"}

    if rank == 0:
        line = {
            "metric": "MoE-layer tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": cfg["dtype"], "data": "synthetic (dyadic tokens/gate, reference demo expert population)",
            "config": {"workload": cfg["workload"], "tokens_per_gpu": T, "hidden": H, "ffn": F, "experts": E,
                       "top_k": k, "sf": sf, "sed": sed, "layers": cfg["layers"], "sr_migration": use_sr,
                       "e2e_host_threads": f"bound to {len(numa_cpus)} GPU-local cores (NVML affinity)" if numa_cpus else "unbound",
                       "clock_ramp": "200 ms of torch bf16 matmul before the warm-up steps",
                       "planner_p": p_plan, "sed_source": sed_source,
                       "planner_mode": (planner or {}).get("mode", "reference model") if p_plan is not None else None, "comm": "none (one GPU)" if world == 1 else ("nccl" if os.environ.get("HEP_COMM") == "nccl" else "nvlink-p2p"),
                       "l2": "inputs larger than L2 (x %.0f MB, expert weights %.2f GB per GPU)" %
                             (T * row_bytes / 1e6, cfg["layers"] * len(layer.owned_experts()) * 2 * H * F * (row_bytes // H) / 1e9)},
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": T * row_bytes,
                    "d2h_bytes_per_step": T * row_bytes},
            "roofline": {"bound": "tensor", "kernel": gemm_kernel,
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per up+down launch pair (ncu, profiles/ncu_summary.json)",
                         "peak_source": peak_source, "peak_burst": peak_burst,
                         "frac_burst": (achieved / peak_burst) if achieved else None,
                         "gemm_ms_per_step": gemm_ms, "timed_in": "the value pass (events around the GEMM launches)",
                         "flops_per_launch_pair": flops / cfg["layers"]},
            "kernels": kernels,
            "planner": planner,
            "gemm_rows_per_gpu": rows_per_gpu,
            "layer_load_imbalance": layer_imbalance,
            "step_ms": step_spread,
            "phase_ms": phases,
            "phase_ms_source": "second pass of the same K steps with events at every phase boundary",
            "gpu_launches": launches,
            "comm": comm_stats,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    for layer in layers:
        layer.close()
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
