"""MoE-layer step (hybridep::moe) over the C-ABI: the drop-in for the step the
reference simulates (sim::build_schedule, simcore.cpp:96-266).

    layer = MoELayer(hidden=4096, ffn=14336, experts=8, top_k=2, max_tokens=16384,
                     dtype=torch.bfloat16, sf=[2, 4], sed=[1, 4], rank=r, comm=comm)
    layer.set_gate(w_gate)                    # H x E
    layer.set_expert(e, w_up, w_down)         # owned experts, reference layout
    layer.gather_experts()                    # expert-domain All-Gather (dense or SR)
    y = layer.forward(x)                      # [T, H] -> [T, H]

Communication is NCCL inside libhep.so; `Communicator.from_torch()` only uses
torch.distributed to broadcast the NCCL unique id.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from ._lib import HEP_BF16, HEP_F32, LayerParams, Level, SrConfig, check, lib
from .sr import CompressionConfig


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dt(dtype) -> int:
    return {torch.float32: HEP_F32, torch.bfloat16: HEP_BF16}[dtype]


class Communicator:
    def __init__(self, handle, rank: int, nranks: int):
        self.handle, self.rank, self.nranks = handle, rank, nranks

    @staticmethod
    def from_torch(group=None) -> "Communicator":
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            check(lib.hep_comm_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        check(lib.hep_comm_init(uid, rank, world, C.byref(h)))
        return Communicator(h, rank, world)

    @staticmethod
    def virtual(nranks: int) -> list:
        """`nranks` virtual ranks on the current device (hep_comm_init_virtual): one
        process drives every rank's layer, each on its own stream."""
        hs = (C.c_void_p * nranks)()
        check(lib.hep_comm_init_virtual(nranks, hs))
        return [Communicator(C.c_void_p(hs[r]), r, nranks) for r in range(nranks)]

    def close(self):
        if self.handle:
            check(lib.hep_comm_destroy(self.handle))
            self.handle = None


def gather_all(layers, stream=None):
    """Queue the expert All-Gather of every layer of a stack at the start of an iteration
    (hep_layers_gather): pulls run in layer order under the compute, each forward waits
    only for its own layer's experts."""
    arr = (C.c_void_p * len(layers))(*[layer.handle.value for layer in layers])
    check(lib.hep_layers_gather(arr, len(layers), _stream(stream)))


class MoELayer:
    def __init__(self, *, hidden, ffn, experts, top_k, max_tokens, dtype=torch.bfloat16, sf=(1,), sed=None,
                 rank=0, comm: Optional[Communicator] = None, sr: Optional[CompressionConfig] = None):
        sed = list(sed) if sed is not None else [1] * len(sf)
        self.H, self.F, self.E, self.k, self.Tmax = hidden, ffn, experts, top_k, max_tokens
        self.dtype, self.sf, self.sed, self.rank = dtype, list(sf), sed, rank
        self.G = 1
        for s in sf:
            self.G *= s
        self.n = experts // self.G
        self._levels = (Level * len(sf))(*[Level(a, b, 1e9) for a, b in zip(sf, sed)])
        srcfg = sr._c() if sr is not None else SrConfig(1.0, -1, 32, 32, 0)
        prm = LayerParams(hidden, ffn, experts, top_k, max_tokens, _dt(dtype), self._levels, len(sf), rank,
                          1 if sr is not None else 0, srcfg)
        self.handle = C.c_void_p()
        check(lib.hep_layer_create(C.byref(prm), comm.handle if comm else None, C.byref(self.handle)))

    def close(self):
        if getattr(self, "handle", None):
            lib.hep_layer_destroy(self.handle)
            self.handle = None

    __del__ = close

    def owned_experts(self):
        return range(self.rank * self.n, (self.rank + 1) * self.n)

    def set_gate(self, w_gate: torch.Tensor, stream=None):
        w_gate = w_gate.contiguous()
        check(lib.hep_layer_set_gate(self.handle, w_gate.data_ptr(), _dt(w_gate.dtype), _stream(stream)))

    def set_expert(self, e: int, w_up: torch.Tensor, w_down: torch.Tensor, stream=None):
        w_up, w_down = w_up.contiguous(), w_down.contiguous()
        check(lib.hep_layer_set_expert(self.handle, e, w_up.data_ptr(), w_down.data_ptr(), _dt(w_up.dtype),
                                       _stream(stream)))

    def set_shared(self, shared_flat_f32: torch.Tensor, stream=None):
        check(lib.hep_layer_set_shared(self.handle, shared_flat_f32.data_ptr(), _stream(stream)))

    def refresh_shared(self, stream=None):
        """Shared expert := mean of all E experts across the ranks (collective; bit-exact
        with the reference's init_shared / update_shared, sparsecomp.cpp:147-173)."""
        check(lib.hep_layer_refresh_shared(self.handle, _stream(stream)))

    def sgd_step(self, grads, lr: float, stream=None):
        """SR mode: SGD step of the owned fp32 masters fused with their migration encode
        (hep_layer_sgd_step); grads: one flat fp32 [2HF] device tensor per owned expert."""
        grads = [g.contiguous() for g in grads]
        arr = (C.c_void_p * len(grads))(*[g.data_ptr() for g in grads])
        check(lib.hep_layer_sgd_step(self.handle, arr, len(grads), float(lr), _stream(stream)))
        self._keep = grads  # alive until the stream reaches the step

    def get_shared(self, stream=None) -> torch.Tensor:
        out = torch.empty(2 * self.H * self.F, dtype=torch.float32, device="cuda")
        check(lib.hep_layer_get_shared(self.handle, out.data_ptr(), _stream(stream)))
        return out

    def gather_experts(self, stream=None):
        check(lib.hep_layer_gather_experts(self.handle, _stream(stream)))

    def forward(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None,
                residual: bool = False) -> torch.Tensor:
        """y = MoE(x); with residual=True, y = x + MoE(x) (the add fused into the combine)."""
        assert x.is_cuda and x.dtype == self.dtype and x.shape[-1] == self.H and x.is_contiguous()
        T = x.shape[0]
        y = out if out is not None else torch.empty_like(x)
        fn = lib.hep_layer_forward_residual if residual else lib.hep_layer_forward
        check(fn(self.handle, x.data_ptr(), T, y.data_ptr(), _stream(stream)))
        return y

    __call__ = forward

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor, stream=None):
        """End-to-end call with host buffers (pinned recommended).  Asynchronous and
        double-buffered; y_host is complete after host_fence() + stream sync."""
        check(lib.hep_layer_forward_host(self.handle, x_host.data_ptr(), x_host.shape[0], y_host.data_ptr(),
                                         _stream(stream)))

    def host_fence(self, stream=None):
        check(lib.hep_layer_host_fence(self.handle, _stream(stream)))

    def check(self, stream=None):
        """Synchronise and raise RuntimeFailure if a migrated expert's wire was rejected."""
        check(lib.hep_layer_check(self.handle, _stream(stream)))

    def debug_corrupt_next_gather(self):
        check(lib.hep_layer_debug_corrupt_next_gather(self.handle))

    def comm_bench(self, x: torch.Tensor, iters: int = 10, stream=None) -> dict:
        """Per-GPU exchange microbenchmark (collective): NVLink A2A dispatch and expert
        All-Gather bytes and times; bus GB/s = bytes / time."""
        out = (C.c_double * 6)()
        check(lib.hep_layer_comm_bench(self.handle, x.data_ptr(), x.shape[0], iters, out, _stream(stream)))
        r = {"a2a_ms": out[0], "a2a_bytes": out[1], "ag_ms": out[3], "ag_bytes": out[4], "ag_pull_ms": out[5]}
        r["a2a_bus_gbs"] = r["a2a_bytes"] / (r["a2a_ms"] * 1e6) if r["a2a_ms"] > 0 else None
        r["ag_bus_gbs"] = r["ag_bytes"] / (r["ag_ms"] * 1e6) if r["ag_ms"] > 0 else None
        # the NVLink transfer of the All-Gather alone (no encode / decode / flags)
        r["ag_pull_bus_gbs"] = r["ag_bytes"] / (r["ag_pull_ms"] * 1e6) if r["ag_pull_ms"] > 0 else None
        return r

    def debug(self, T: int):
        """Device views of the last forward's routing: topk_idx, topk_w, pos, key_counts."""
        ti, tw, pos, packed, kc = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib.hep_layer_debug(self.handle, C.byref(ti), C.byref(tw), C.byref(pos), C.byref(packed), C.byref(kc)))
        dev = torch.cuda.current_device()

        def view(ptr, n, dtype):
            class _Dev:  # zero-copy view of layer-owned device memory, then an owned copy
                __cuda_array_interface__ = {"shape": (n,), "version": 3, "data": (ptr.value, False),
                                            "typestr": {torch.int32: "<i4", torch.float32: "<f4",
                                                        torch.bfloat16: "<u2"}[dtype]}
            t = torch.as_tensor(_Dev(), device=dev).clone()
            return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t

        kT = T * self.k
        rows = kT  # packed send rows of this GPU
        return {
            "topk_idx": view(ti, kT, torch.int32).view(T, self.k),
            "topk_w": view(tw, kT, torch.float32).view(T, self.k),
            "pos": view(pos, kT, torch.int32).view(T, self.k),
            "packed": view(packed, rows * self.H, self.dtype).view(rows, self.H),
            "key_counts": view(kc, self.G * self.E, torch.int32),
        }

    def set_profiling(self, level):
        """0/False off, 1 events around the expert GEMMs only, 2/True every phase."""
        level = 2 if level is True else int(level)
        check(lib.hep_layer_set_profiling(self.handle, level))

    def timings(self) -> dict:
        names = C.create_string_buffer(1024)
        ms = (C.c_float * 32)()
        cnt = C.c_int()
        check(lib.hep_layer_timings(self.handle, names, 1024, ms, 32, C.byref(cnt)))
        keys = names.value.decode().split(";") if cnt.value else []
        return dict(zip(keys, list(ms)[: cnt.value]))

    def gemm_schedule(self) -> tuple:
        """(up, down) L2-policy/raster words of the bf16 expert GEMMs (hep_grouped_gemm sched)."""
        u, d = C.c_uint32(), C.c_uint32()
        check(lib.hep_layer_gemm_schedule(self.handle, C.byref(u), C.byref(d)))
        return u.value, d.value

    def launch_count(self) -> int:
        c = C.c_int()
        check(lib.hep_layer_launch_count(self.handle, C.byref(c)))
        return c.value
