"""The "cuda" backend: the reference backend interface over libslicegemm_b200.so.

Mirrors slicegemm/_core_py.py (the "pure" backend, selected through _core.py:15-61): the same
function names and in-place semantics, argument order destination planes low to high then
source planes (_core_py.py:8-9).  Arrays are per-plane (rows, words) 64-bit word arrays:
CUDA torch tensors (int64 or uint64 bit patterns) are updated in place on the device; numpy
uint64 arrays are accepted too (copied to the GPU, updated, copied back) so a caller written
against the pure backend runs unchanged.  The whole-product entry point m4rm_multiply (one
launch sequence for all k-blocks) is the fast path; these block-granularity calls exist for
interface parity (one launch per call).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

NAME = "cuda"


def _as_dev(arrs):
    """Return device tensors for arrs, plus a write-back closure for numpy inputs."""
    devs, backs = [], []
    for a in arrs:
        if isinstance(a, torch.Tensor):
            if a.device.type != "cuda":
                raise ValueError("cuda backend: tensors must live on a CUDA device")
            t = a if a.dtype == torch.int64 else a.view(torch.int64)
            if not t.is_contiguous():
                raise ValueError("cuda backend: plane arrays must be contiguous")
            devs.append(t)
            backs.append(None)
        else:
            arr = np.asarray(a)
            if arr.dtype != np.uint64:
                raise ValueError("cuda backend: plane arrays must be uint64")
            t = torch.from_numpy(np.ascontiguousarray(arr).view(np.int64)).cuda()
            devs.append(t)
            backs.append(arr)
    return devs, backs


def _write_back(devs, backs):
    for t, arr in zip(devs, backs):
        if arr is not None:
            arr[...] = t.cpu().numpy().view(np.uint64).reshape(arr.shape)


def _shape(t):
    return (1, t.shape[0]) if t.dim() == 1 else (t.shape[0], t.shape[1])


def _op(name, dst, src=(), tail=(1 << 64) - 1, scalar=0):
    d, db = _as_dev(dst)
    s, _ = _as_dev(src)
    rows, words = _shape(d[0])
    dp, _k1 = _lib.ptr_array([t.data_ptr() for t in d])
    sp, _k2 = _lib.ptr_array([t.data_ptr() for t in s]) if s else (None, None)
    with torch.cuda.device(d[0].device):
        _lib.check(_lib.load().sg_plane_op(_lib.OPS[name], dp, sp, rows, words, int(tail) & ((1 << 64) - 1),
                                           scalar, _lib.current_stream_handle(d[0].device)))
    _write_back(d, db)


def f2_add(d0, s0): _op("f2_add", [d0], [s0])
def f3_add(d0, d1, s0, s1): _op("f3_add", [d0, d1], [s0, s1])
def f3_sub(d0, d1, s0, s1): _op("f3_sub", [d0, d1], [s0, s1])
def f3_neg(p0, p1): _op("f3_neg", [p0, p1])
def f5_add(d0, d1, d2, s0, s1, s2): _op("f5_add", [d0, d1, d2], [s0, s1, s2])
def f5_sub(d0, d1, d2, s0, s1, s2): _op("f5_sub", [d0, d1, d2], [s0, s1, s2])
def f5_neg(p0, p1, p2): _op("f5_neg", [p0, p1, p2])
def f5_double(p0, p1, p2): _op("f5_double", [p0, p1, p2])
def f5_reduce(p0, p1, p2): _op("f5_reduce", [p0, p1, p2])
def f7_add(d0, d1, d2, s0, s1, s2): _op("f7_add", [d0, d1, d2], [s0, s1, s2])
def f7_sub(d0, d1, d2, s0, s1, s2, tail): _op("f7_sub", [d0, d1, d2], [s0, s1, s2], tail=tail)
def f7_neg(p0, p1, p2, tail): _op("f7_neg", [p0, p1, p2], tail=tail)
def f7_reduce(p0, p1, p2): _op("f7_reduce", [p0, p1, p2])
def z4_add(d0, d1, s0, s1): _op("z4_add", [d0, d1], [s0, s1])
def z4_sub(d0, d1, s0, s1): _op("z4_sub", [d0, d1], [s0, s1])
def z4_neg(p0, p1): _op("z4_neg", [p0, p1])
def z8_add(d0, d1, d2, s0, s1, s2): _op("z8_add", [d0, d1, d2], [s0, s1, s2])
def z8_sub(d0, d1, d2, s0, s1, s2): _op("z8_sub", [d0, d1, d2], [s0, s1, s2])
def z8_neg(p0, p1, p2): _op("z8_neg", [p0, p1, p2])


def _block(field_code, C, A, col0, kp, T, row0, row1):
    c, cb = _as_dev(C)
    a, _ = _as_dev(A)
    t, _ = _as_dev(T)
    (crows, cw), (arows, aw) = _shape(c[0]), _shape(a[0])
    # the reference block driver indexes numpy arrays and raises IndexError / ValueError on these
    # (_core_py.py:205-281); here they would be out-of-bounds device accesses, so check first
    for group, what in ((c, "C"), (a, "A"), (t, "T")):
        if any(_shape(x) != _shape(group[0]) for x in group):
            raise ValueError(f"{what} planes differ in shape")
    row0, row1, col0, kp = int(row0), int(row1), int(col0), int(kp)
    if not 0 <= row0 <= row1 <= crows or row1 > arows:
        raise IndexError(f"rows [{row0}, {row1}) outside C ({crows} rows) or A ({arows} rows)")
    if kp < 0 or col0 < 0 or col0 + kp > 64 * aw:
        raise IndexError(f"block columns [{col0}, {col0 + kp}) outside A ({64 * aw} columns)")
    trows, tw = _shape(t[0])
    if row1 > row0 and kp > 0 and trows < (1 << kp):
        raise IndexError(f"table has {trows} entries, block needs {1 << kp}")
    if tw != cw:
        raise ValueError(f"table rows have {tw} words, C rows {cw}")
    cp, _k1 = _lib.ptr_array([x.data_ptr() for x in c])
    ap, _k2 = _lib.ptr_array([x.data_ptr() for x in a])
    tp, _k3 = _lib.ptr_array([x.data_ptr() for x in t])
    with torch.cuda.device(c[0].device):
        _lib.check(_lib.load().sg_m4rm_block(field_code, cp, cw, ap, aw, int(col0), int(kp), tp, int(row0),
                                             int(row1), _lib.current_stream_handle(c[0].device)))
    _write_back(c, cb)


def m4rm_block_f2(C0, A0, col0, kp, T0, row0, row1):
    _block(_lib.SG_F2, [C0], [A0], col0, kp, [T0], row0, row1)


def m4rm_block_f3(C0, C1, A0, A1, col0, kp, T0, T1, row0, row1):
    _block(_lib.SG_F3, [C0, C1], [A0, A1], col0, kp, [T0, T1], row0, row1)


def m4rm_block_f5(C0, C1, C2, A0, A1, A2, col0, kp, T0, T1, T2, row0, row1):
    _block(_lib.SG_F5, [C0, C1, C2], [A0, A1, A2], col0, kp, [T0, T1, T2], row0, row1)


def m4rm_block_f7(C0, C1, C2, A0, A1, A2, col0, kp, T0, T1, T2, row0, row1):
    _block(_lib.SG_F7, [C0, C1, C2], [A0, A1, A2], col0, kp, [T0, T1, T2], row0, row1)


def m4rm_block_gf4(C0, C1, A0, A1, col0, kp, T0, T1, row0, row1):
    _block(_lib.SG_GF4, [C0, C1], [A0, A1], col0, kp, [T0, T1], row0, row1)


def m4rm_block_gf8(C0, C1, C2, A0, A1, A2, col0, kp, T0, T1, T2, row0, row1):
    _block(_lib.SG_GF8, [C0, C1, C2], [A0, A1, A2], col0, kp, [T0, T1, T2], row0, row1)


def m4rm_block_z4(C0, C1, A0, A1, col0, kp, T0, T1, row0, row1):
    _block(_lib.SG_Z4, [C0, C1], [A0, A1], col0, kp, [T0, T1], row0, row1)


def m4rm_block_z8(C0, C1, C2, A0, A1, A2, col0, kp, T0, T1, T2, row0, row1):
    _block(_lib.SG_Z8, [C0, C1, C2], [A0, A1, A2], col0, kp, [T0, T1, T2], row0, row1)


# ---------------------------------------------------------------- classical drivers
def _classical(field_code, C, A, B):
    """C += A B in place with the pure backend's raw row-accumulate semantics (_core_py.py:292-366)."""
    c, cb = _as_dev(C)
    a, _ = _as_dev(A)
    b, _ = _as_dev(B)
    (m, cw), (arows, aw), (l, bw) = _shape(c[0]), _shape(a[0]), _shape(b[0])
    for group, what in ((c, "C"), (a, "A"), (b, "B")):
        if any(_shape(x) != _shape(group[0]) for x in group):
            raise ValueError(f"{what} planes differ in shape")
    if arows != m:
        raise ValueError(f"A has {arows} rows, C {m}")
    if bw != cw:
        raise ValueError(f"B rows have {bw} words, C rows {cw}")
    if l > 64 * aw:
        raise IndexError(f"B has {l} rows but A only {64 * aw} columns")
    cp, _k1 = _lib.ptr_array([x.data_ptr() for x in c])
    ap, _k2 = _lib.ptr_array([x.data_ptr() for x in a])
    bp, _k3 = _lib.ptr_array([x.data_ptr() for x in b])
    with torch.cuda.device(c[0].device):
        _lib.check(_lib.load().sg_classical_block(field_code, cp, cw, ap, aw, bp, m, l,
                                                  _lib.current_stream_handle(c[0].device)))
    _write_back(c, cb)


def classical_f2(C0, A0, B0):
    _classical(_lib.SG_F2, [C0], [A0], [B0])


def classical_f3(C0, C1, A0, A1, B0, B1):
    _classical(_lib.SG_F3, [C0, C1], [A0, A1], [B0, B1])


def classical_z4(C0, C1, A0, A1, B0, B1):
    _classical(_lib.SG_Z4, [C0, C1], [A0, A1], [B0, B1])


def classical_f5(C0, C1, C2, A0, A1, A2, B0, B1, B2):
    _classical(_lib.SG_F5, [C0, C1, C2], [A0, A1, A2], [B0, B1, B2])


def classical_f7(C0, C1, C2, A0, A1, A2, B0, B1, B2):
    _classical(_lib.SG_F7, [C0, C1, C2], [A0, A1, A2], [B0, B1, B2])


def classical_z8(C0, C1, C2, A0, A1, A2, B0, B1, B2):
    _classical(_lib.SG_Z8, [C0, C1, C2], [A0, A1, A2], [B0, B1, B2])


# Names of the pure backend (_core_py.py) this module deliberately does not provide: the
# packed-integer baselines (_core_py.py:372-380) and the program-search engine
# (_core_py.py:381-661) are outside the M4RM hot path.
OUT_OF_SCOPE = ("packed_z4_add", "packed_f3_add", "run_exhaustive", "run_staged")
