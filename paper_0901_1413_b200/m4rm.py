"""m4rm_multiply and friends: the reference multiply API over the B200 kernels.

Contract: SPEC.md:301-367 (the reference's m4rm.py is missing; names from __init__.py:16).
  M4rmParams(k)        SPEC.md:306-311   (1 <= k <= 16)
  choose_k(l)          SPEC.md:340-346   clamp(floor(log2 l) - 2, 1, 10)
  build_table(B, s, k) SPEC.md:313-325   mask-indexed table of one k-row block of B
  m4rm_multiply(A, B)  SPEC.md:326-332   C = A B, equal to the oracle after canonicalization;
                                          this implementation returns C canonical and
                                          bit-identical for every k (k > 8 uses 8-row blocks).
Device matrices run sg_m4rm on the current CUDA stream; two host matrices run the
host-buffer entry point sg_m4rm_host (H2D, multiply, D2H).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .matrix import BitslicedMatrix, _require_cuda, _vp


@dataclass(frozen=True)
class M4rmParams:
    k: int = None

    def __post_init__(self):
        if self.k is not None and not 1 <= self.k <= 16:
            raise ValueError("k must be in 1..16")


def choose_k(l: int) -> int:
    if l < 1:
        return 1
    return max(1, min(10, l.bit_length() - 1 - 2))


def _check(A: BitslicedMatrix, B: BitslicedMatrix):
    if not isinstance(A, BitslicedMatrix) or not isinstance(B, BitslicedMatrix):
        raise TypeError("m4rm_multiply takes two BitslicedMatrix operands")
    if A.field is not B.field:
        raise ValueError(f"field mismatch: {A.field.name} vs {B.field.name}")
    if A.ncols != B.nrows:
        raise ValueError(f"inner dimensions {A.ncols} != {B.nrows}")


def m4rm_multiply(A: BitslicedMatrix, B: BitslicedMatrix, params: M4rmParams = None,
                  out: BitslicedMatrix = None) -> BitslicedMatrix:
    _check(A, B)
    k = (params.k if params is not None and params.k is not None else None) or choose_k(A.ncols)
    m, l, n = A.nrows, A.ncols, B.ncols
    field = A.field
    L = _lib.load()
    if A.device.type == "cpu" and B.device.type == "cpu":
        # host buffers in, host buffers out: the reference-facing call with copies included
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device is available: the B200 path has no CPU fallback")
        a = A.planes.contiguous()
        b = B.planes.contiguous()
        if out is None:
            if a.is_pinned() and b.is_pinned():  # page-locked in, page-locked out: async copies
                C = BitslicedMatrix.pinned_empty(field, m, n) if m and n and l else BitslicedMatrix.pinned_zero(field, m, n)
            else:
                # every word of C (padding lanes included) comes down from the device: no need to
                # zero 8 R m W bytes of fresh pageable memory first
                alloc = torch.empty if (m and n and l) else torch.zeros  # (an empty product writes nothing)
                C = BitslicedMatrix(field, m, n, alloc((field.bits, m, (n + 63) // 64), dtype=torch.int64))
        else:
            # sg_m4rm_host writes R*m*W words through this pointer: the same checks as on the
            # device, plus host residency (a device pointer is not a host buffer)
            if not isinstance(out, BitslicedMatrix) or out.field is not field or (out.nrows, out.ncols) != (m, n):
                raise ValueError("out has the wrong field or shape")
            if out.device.type != "cpu":
                raise ValueError("out must be a host matrix when both operands are on the host")
            if not out.planes.is_contiguous():
                out.planes = out.planes.contiguous()
            for t in (a, b):
                lo, hi = t.data_ptr(), t.data_ptr() + t.numel() * 8
                if t.numel() and out.planes.numel() and lo < out.planes.data_ptr() + out.planes.numel() * 8 \
                        and out.planes.data_ptr() < hi:
                    raise ValueError("out must not overlap the operands")
            C = out
        if m and n:
            _lib.check(L.sg_m4rm_host(field.code, _vp(a), _vp(b), _vp(C.planes), m, l, n, k,
                                      torch.cuda.current_device()))
        return C
    dev = A.device if A.device.type == "cuda" else B.device
    _require_cuda(dev)
    a = A.planes if A.planes.device == dev else A.planes.to(dev).contiguous()
    b = B.planes if B.planes.device == dev else B.planes.to(dev).contiguous()
    if out is None:
        C = BitslicedMatrix(field, m, n, torch.empty((field.bits, m, (n + 63) // 64), dtype=torch.int64, device=dev))
    else:
        if out.field is not field or (out.nrows, out.ncols) != (m, n) or out.device != dev:
            raise ValueError("out has the wrong field, shape or device")
        for t in (a, b):  # the kernels read A and B while C is written
            lo, hi = t.data_ptr(), t.data_ptr() + t.numel() * 8
            if t.numel() and out.planes.numel() and lo < out.planes.data_ptr() + out.planes.numel() * 8 \
                    and out.planes.data_ptr() < hi:
                raise ValueError("out must not overlap the operands")
        C = out
    if m and n:
        if dev.index == torch.cuda.current_device():  # the common case: no device switch
            _lib.check(L.sg_m4rm(field.code, _vp(a), _vp(b), _vp(C.planes), m, l, n, k, None, 0,
                                 _lib.current_stream_handle(dev)))
        else:
            with torch.cuda.device(dev):
                _lib.check(L.sg_m4rm(field.code, _vp(a), _vp(b), _vp(C.planes), m, l, n, k, None, 0,
                                     _lib.current_stream_handle(dev)))
    return C


def classical_multiply(A: BitslicedMatrix, B: BitslicedMatrix) -> BitslicedMatrix:
    """C = A B by row accumulation without tables: the reference's mid-level
    cross-check, on the GPU (O(m l n / 32) word operations)."""
    _check(A, B)
    m, l, n = A.nrows, A.ncols, B.ncols
    dev = A.device if A.device.type == "cuda" else B.device
    if dev.type != "cuda":
        dev = torch.device("cuda", torch.cuda.current_device())
    _require_cuda(dev)
    a, b = A.planes.to(dev).contiguous(), B.planes.to(dev).contiguous()
    C = BitslicedMatrix(A.field, m, n, torch.empty((A.field.bits, m, (n + 63) // 64), dtype=torch.int64, device=dev))
    if m and n:
        with torch.cuda.device(dev):
            _lib.check(_lib.load().sg_classical(A.field.code, _vp(a), _vp(b), _vp(C.planes), m, l, n,
                                                _lib.current_stream_handle(dev)))
    return C


def build_table(B: BitslicedMatrix, s: int, k: int) -> torch.Tensor:
    """Table of block s (rows s*k .. s*k+kp-1 of B): int64 tensor (R, 2^kp, words).

    Entry g is the field sum of the rows whose bit is set in g (so T[0] = 0); the final block
    may be narrower (kp = l - s*k).
    """
    if not 1 <= k <= 16:
        raise ValueError("k must be in 1..16")
    l = B.nrows
    if not 0 <= s * k < max(l, 1):
        raise ValueError("block index out of range")
    kp = min(k, l - s * k)
    Bg = B._on_gpu()
    R, W = B.field.bits, B.words_per_row
    T = torch.zeros((R, 1 << kp, W), dtype=torch.int64, device=Bg.device)
    bp, _k1 = _lib.ptr_array([Bg.planes[d].data_ptr() for d in range(R)])
    tp, _k2 = _lib.ptr_array([T[d].data_ptr() for d in range(R)])
    with torch.cuda.device(Bg.device):
        _lib.check(_lib.load().sg_build_table(B.field.code, bp, l, s * k, kp, W, tp,
                                              _lib.current_stream_handle(Bg.device)))
    return T


SCHEDULES = {0: "serial", 1: "pipelined", 2: "warp-specialized (4 builder warps)",
             3: "warp-specialized (1 builder warp)", 4: "warp-specialized (2 builder warps)",
             5: "warp-specialized (8 builder warps)",
             6: "warp-specialized (4 builder warps, TMEM row-slots)",
             10: "fused serial (one launch)", 11: "fused pipelined (one launch)"}
# schedule codes of the fused small-product variants (sg_set_plan_override's `pipe`)
FUSED_SERIAL, FUSED_PIPELINED = 10, 11


def plan(field, m: int, l: int, n: int, k: int = 8) -> dict:
    """The launch the planner picks for this product (rows per CTA, k-splits, CTAs)."""
    from .fields import by_name
    if isinstance(field, str):
        field = by_name(field)
    rows, splits, ctas, idx, pipe, thr = (ctypes.c_int() for _ in range(6))
    _lib.check(_lib.load().sg_plan(field.code, m, l, n, k, ctypes.byref(rows), ctypes.byref(splits),
                                   ctypes.byref(ctas), ctypes.byref(idx), ctypes.byref(pipe), ctypes.byref(thr)))
    return {"rows_per_cta": rows.value, "splits": splits.value, "ctas": ctas.value, "kernel": idx.value,
            "schedule": SCHEDULES.get(pipe.value, str(pipe.value)), "threads": thr.value}


def set_plan_override(rows_per_thread: int = 0, splits: int = 0, pipe: int = -1, threads: int = 0):
    _lib.check(_lib.load().sg_set_plan_override(rows_per_thread, splits, pipe, threads))


def set_sm_reserve(sms: int = 0):
    """Leave `sms` SMs free in subsequent plans (for a concurrent collective); 0 = use all."""
    _lib.check(_lib.load().sg_set_sm_reserve(sms))


def last_timing() -> dict:
    t, mm, r = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.load().sg_last_timing(ctypes.byref(t), ctypes.byref(mm), ctypes.byref(r)))
    return {"transpose_ms": t.value, "m4rm_ms": mm.value, "reduce_ms": r.value}


def set_timing(enable: bool):
    _lib.check(_lib.load().sg_set_timing(1 if enable else 0))


def kernel_info(device: int = 0) -> list:
    """Every compiled M4RM instantiation: field code, k, rows per thread, lookup threads,
    schedule, CTAs per SM, registers per thread, dynamic shared memory bytes."""
    L = _lib.load()
    out, i = [], 0
    while True:
        v = [ctypes.c_int() for _ in range(8)]
        n = L.sg_kernel_info(i, device, *(ctypes.byref(x) for x in v))
        if n < 0:
            return out
        out.append(dict(zip(("field", "k", "rt", "threads", "schedule", "occupancy", "regs", "smem_bytes"),
                            (x.value for x in v)), index=i))
        i += 1


def launch_count() -> int:
    return int(_lib.load().sg_launch_count())


def probe_peaks(device: int = 0) -> dict:
    a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.load().sg_probe_peaks(device, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return {"lop3_per_clk_per_sm": a.value, "lds_bytes_per_clk_per_sm": b.value, "sm_mhz": c.value}
