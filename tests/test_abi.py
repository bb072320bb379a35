"""CPU tests of the C ABI boundary: the library loads and exports every declared symbol,
and argument validation answers without touching a GPU."""

import ctypes
import os
import re

import pytest

from paper_0901_1413_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for name in os.listdir(inc):
        if name.endswith(".h"):
            text = open(os.path.join(inc, name)).read()
            syms |= set(re.findall(r"\b(sg_\w+)\s*\(", text))
    return syms


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 18
    assert syms == set(_lib.EXPORTS)
    for s in syms:
        assert getattr(L, s) is not None
    # no result-corrupting experiment switch in the production library
    assert not hasattr(L, "sg_debug_ablation")


def test_abi_version_and_planes():
    L = _lib.load()
    assert L.sg_abi_version() == 1
    assert [L.sg_field_planes(f) for f in range(8)] == [1, 2, 3, 3, 2, 3, 2, 3]
    assert L.sg_field_planes(9) == -1


def test_invalid_arguments_are_rejected_before_cuda():
    L = _lib.load()
    vp = ctypes.c_void_p
    rc = L.sg_m4rm(99, vp(1), vp(1), vp(1), 4, 4, 4, 8, None, 0, None)
    assert rc == _lib.SG_EINVAL and b"field" in L.sg_last_error()
    rc = L.sg_m4rm(1, vp(1), vp(1), vp(1), 4, 4, 4, 0, None, 0, None)
    assert rc == _lib.SG_EINVAL and b"k must be" in L.sg_last_error()
    rc = L.sg_m4rm(1, None, vp(1), vp(1), 4, 4, 4, 8, None, 0, None)
    assert rc == _lib.SG_EINVAL
    rc = L.sg_m4rm(1, vp(1), vp(1), vp(1), -1, 4, 4, 8, None, 0, None)
    assert rc == _lib.SG_EINVAL
    assert L.sg_plane_op(99, None, None, 1, 1, 0, 0, None) == _lib.SG_EINVAL
    assert L.sg_kernel_info(-1, 0, None, None, None, None, None, None, None, None) == -1
    # C overlapping an operand is rejected before any device work
    assert L.sg_m4rm(1, vp(4096), vp(1 << 20), vp(4096 + 64), 8, 8, 8, 8, None, 0, None) == _lib.SG_EINVAL
    assert b"overlaps" in L.sg_last_error()
    assert L.sg_pack(1, None, 2, 5, 3, None, None) == _lib.SG_EINVAL  # ld < n
    with pytest.raises(ValueError):
        _lib.check(_lib.SG_EINVAL)
    with pytest.raises(_lib.SliceGemmError):
        _lib.check(_lib.SG_ECUDA)


def test_empty_products_are_no_ops():
    L = _lib.load()
    assert L.sg_m4rm(1, None, None, None, 0, 5, 5, 8, None, 0, None) == _lib.SG_OK
    assert L.sg_m4rm(1, None, None, None, 5, 5, 0, 8, None, 0, None) == _lib.SG_OK
