"""Device SR migration codec (pack/unpack) — Python mirror of hybridep::sr
(proj/include/hybridep/sparsecomp.hpp) over the C-ABI.

Tensors are torch CUDA tensors (torch is only the allocator here); every call runs
the sm_100a kernels in libhep.so on the current stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from ._lib import HEP_BF16, HEP_F32, SrConfig, check, lib

WIRE_HEADER_BYTES = 28


@dataclass
class CompressionConfig:
    ratio_CR: Optional[float] = None
    k: Optional[int] = None
    index_width_bits: int = 32
    value_width_bits: int = 32
    per_matrix_budget: bool = False

    def _c(self) -> SrConfig:
        return SrConfig(float(self.ratio_CR or 1.0), -1 if self.k is None else int(self.k),
                        self.index_width_bits, self.value_width_bits, int(self.per_matrix_budget))

    def resolve_k(self, total_elements: int, element_width_bytes: int = 4) -> int:
        if self.k is None and self.ratio_CR is None:
            from ._lib import InvalidArgument
            raise InvalidArgument(2, "compression config needs a ratio or a k")
        k = C.c_int64()
        check(lib.hep_sr_resolve_k(C.byref(self._c()), total_elements, element_width_bytes, C.byref(k)))
        return k.value


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return HEP_F32
    if t.dtype == torch.bfloat16:
        return HEP_BF16
    raise TypeError(f"unsupported dtype {t.dtype}")


def wire_bytes(h: int, m: int, cfg: CompressionConfig) -> int:
    n = C.c_size_t()
    check(lib.hep_sr_wire_bytes(h, m, C.byref(cfg._c()), C.byref(n)))
    return n.value


_ws_cache: dict = {}


def _workspace(device, h: int, m: int, batch: int = 1) -> torch.Tensor:
    n = C.c_size_t()
    check(lib.hep_sr_workspace_bytes(h, m, batch, C.byref(n)))
    key = str(device)
    if key not in _ws_cache or _ws_cache[key].numel() < n.value:
        _ws_cache[key] = torch.empty(n.value, dtype=torch.uint8, device=device)
    return _ws_cache[key]


def sr_encode(expert: torch.Tensor, shared: torch.Tensor, h: int, m: int, cfg: CompressionConfig) -> torch.Tensor:
    """Flat expert (P = 2hm, fp32/bf16) vs flat fp32 shared -> SRC1 wire (uint8, device)."""
    assert expert.is_cuda and expert.is_contiguous() and shared.dtype == torch.float32
    nbytes = wire_bytes(h, m, cfg)
    wire = torch.empty(nbytes, dtype=torch.uint8, device=expert.device)
    ws = _workspace(expert.device, h, m)
    check(lib.hep_sr_encode(expert.data_ptr(), _dt(expert), shared.data_ptr(), h, m, C.byref(cfg._c()),
                            wire.data_ptr(), nbytes, ws.data_ptr(), ws.numel(), _stream()))
    return wire


def sr_encode_batch(experts: list, shared: torch.Tensor, h: int, m: int, cfg: CompressionConfig) -> list:
    """Encodes several experts (same shape, same shared expert) in one launch sequence."""
    n = len(experts)
    nbytes = wire_bytes(h, m, cfg)
    wires = [torch.empty(nbytes, dtype=torch.uint8, device=shared.device) for _ in range(n)]
    ws = _workspace(shared.device, h, m, n)
    eps = (C.c_void_p * n)(*[e.data_ptr() for e in experts])
    wps = (C.c_void_p * n)(*[w.data_ptr() for w in wires])
    check(lib.hep_sr_encode_batch(eps, n, _dt(experts[0]), shared.data_ptr(), h, m, C.byref(cfg._c()), wps, nbytes,
                                  ws.data_ptr(), ws.numel(), _stream()))
    return wires


def sr_decode_batch(wires: list, shared: torch.Tensor, h: int, m: int, check_status: bool = True) -> list:
    n = len(wires)
    outs = [torch.empty(2 * h * m, dtype=torch.float32, device=shared.device) for _ in range(n)]
    status = torch.zeros(4 * n, dtype=torch.int32, device=shared.device)
    wps = (C.c_void_p * n)(*[w.data_ptr() for w in wires])
    ops = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    check(lib.hep_sr_decode_batch(wps, n, wires[0].numel(), shared.data_ptr(), h, m, ops, status.data_ptr(),
                                  _stream()))
    if check_status:
        for i in range(n):
            check(lib.hep_sr_check_status(status[4 * i:].data_ptr(), _stream()))
    return outs


def sr_decode(wire: torch.Tensor, shared: torch.Tensor, h: int, m: int, check_status: bool = True) -> torch.Tensor:
    """SRC1 wire (device) + flat fp32 shared -> flat fp32 expert.  Raises the
    reference's exception class on a corrupt wire when check_status (syncs)."""
    out = torch.empty(2 * h * m, dtype=torch.float32, device=shared.device)
    status = torch.zeros(4, dtype=torch.int32, device=shared.device)
    check(lib.hep_sr_decode(wire.data_ptr(), wire.numel(), shared.data_ptr(), h, m, out.data_ptr(),
                            status.data_ptr(), _stream()))
    if check_status:
        check(lib.hep_sr_check_status(status.data_ptr(), _stream()))
    return out


def shared_mean(experts: list) -> torch.Tensor:
    """init_shared / update_shared: fp64 mean in list order, rounded to fp32."""
    assert experts
    P = experts[0].numel()
    out = torch.empty(P, dtype=torch.float32, device=experts[0].device)
    ptrs = (C.c_void_p * len(experts))(*[e.data_ptr() for e in experts])
    check(lib.hep_shared_mean(ptrs, len(experts), _dt(experts[0]), P, out.data_ptr(), _stream()))
    return out


def sr_encode_update_batch(masters: list, grads: list, lr: float, shared: torch.Tensor, h: int, m: int,
                           cfg: CompressionConfig) -> list:
    """The optimizer step fused with the encode (hep_sr_encode_update_batch): every fp32
    master (flat P, device) becomes fmaf(-lr, grad, master) IN PLACE and is encoded."""
    n = len(masters)
    nbytes = wire_bytes(h, m, cfg)
    wires = [torch.empty(nbytes, dtype=torch.uint8, device=shared.device) for _ in range(n)]
    ws = _workspace(shared.device, h, m, n)
    mps = (C.c_void_p * n)(*[t.data_ptr() for t in masters])
    gps = (C.c_void_p * n)(*[t.data_ptr() for t in grads])
    wps = (C.c_void_p * n)(*[w.data_ptr() for w in wires])
    check(lib.hep_sr_encode_update_batch(mps, gps, n, lr, shared.data_ptr(), h, m, C.byref(cfg._c()), wps, nbytes,
                                         ws.data_ptr(), ws.numel(), _stream()))
    return wires


def sgd_step_batch(masters: list, grads: list, lr: float):
    """The unfused step: masters[b] = fmaf(-lr, grads[b], masters[b]) in place."""
    n = len(masters)
    mps = (C.c_void_p * n)(*[t.data_ptr() for t in masters])
    gps = (C.c_void_p * n)(*[t.data_ptr() for t in grads])
    check(lib.hep_sgd_step_batch(mps, gps, n, masters[0].numel(), lr, _stream()))
