"""ctypes binding of libslicegemm_b200.so (the C ABI declared in include/slicegemm_b200.h).

There is no fallback: if the library or a CUDA device is missing, every compute entry point
raises.  The library is built in-tree by __graft_entry__.build() (csrc/Makefile).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslicegemm_b200.so")

# field codes (include/slicegemm_b200.h)
SG_F2, SG_F3, SG_F5, SG_F7, SG_GF4, SG_GF8, SG_Z4, SG_Z8 = 0, 1, 2, 3, 4, 5, 6, 7

# status codes
SG_OK, SG_EINVAL, SG_ECUDA, SG_EUNSUPPORTED, SG_ERANGE, SG_EPATTERN, SG_ENOMEM = range(7)

# plane-op codes
OPS = {
    "f2_add": 0, "f3_add": 1, "f3_sub": 2, "f3_neg": 3, "f5_add": 4, "f5_sub": 5, "f5_neg": 6,
    "f5_double": 7, "f5_reduce": 8, "f7_add": 9, "f7_sub": 10, "f7_neg": 11, "f7_double": 12,
    "f7_reduce": 13, "gf4_add": 14, "gf4_mulx": 15, "f5_fold5": 16, "scalar_mul_f3": 17,
    "scalar_mul_f5": 18, "scalar_mul_f7": 19, "scalar_mul_gf4": 20, "z4_add": 21, "z4_sub": 22, "z4_neg": 23,
    "z8_add": 24, "z8_sub": 25, "z8_neg": 26, "gf8_add": 27, "gf8_mulx": 28, "scalar_mul_z4": 29,
    "scalar_mul_z8": 30, "scalar_mul_gf8": 31,
}

# every symbol include/slicegemm_b200.h declares
EXPORTS = (
    "sg_abi_version", "sg_last_error", "sg_field_planes", "sg_pack", "sg_unpack", "sg_stream_check",
    "sg_reduce_canonical", "sg_plane_op", "sg_m4rm_workspace_bytes", "sg_m4rm", "sg_m4rm_host", "sg_m4rm_multi",
    "sg_build_table", "sg_m4rm_block", "sg_plan", "sg_set_plan_override", "sg_set_sm_reserve", "sg_set_timing",
    "sg_last_timing", "sg_launch_count", "sg_host_streamed_count", "sg_kernel_info", "sg_probe_peaks", "sg_classical", "sg_classical_block",
)

_lib = None


class SliceGemmError(RuntimeError):
    pass


def load():
    """Load the library (raises if it is missing: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SG_LIB_PATH", LIB_PATH)  # experiments: A/B against another build
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback for the B200 path)")
    L = ctypes.CDLL(path)
    i64, i32, vp, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64
    pp = ctypes.POINTER(ctypes.c_void_p)
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int)
    sig = {
        "sg_abi_version": ([], i32),
        "sg_last_error": ([], ctypes.c_char_p),
        "sg_field_planes": ([i32], i32),
        "sg_pack": ([i32, vp, i64, i64, i64, vp, vp], i32),
        "sg_unpack": ([i32, vp, i64, i64, vp, i64, vp], i32),
        "sg_stream_check": ([vp], i32),
        "sg_reduce_canonical": ([i32, vp, i64, i64, vp], i32),
        "sg_plane_op": ([i32, pp, pp, i64, i64, u64, i32, vp], i32),
        "sg_m4rm_workspace_bytes": ([i32, i64, i64, i64, i32], i64),
        "sg_m4rm": ([i32, vp, vp, vp, i64, i64, i64, i32, vp, i64, vp], i32),
        "sg_m4rm_host": ([i32, vp, vp, vp, i64, i64, i64, i32, i32], i32),
        "sg_m4rm_multi": ([i32, vp, vp, vp, i64, i64, i64, i32, i32, ip], i32),
        "sg_build_table": ([i32, pp, i64, i64, i32, i64, pp, vp], i32),
        "sg_m4rm_block": ([i32, pp, i64, pp, i64, i64, i32, pp, i64, i64, vp], i32),
        "sg_plan": ([i32, i64, i64, i64, i32, ip, ip, ip, ip, ip, ip], i32),
        "sg_set_plan_override": ([i32, i32, i32, i32], i32),
        "sg_set_sm_reserve": ([i32], i32),
        "sg_set_timing": ([i32], i32),
        "sg_last_timing": ([dp, dp, dp], i32),
        "sg_launch_count": ([], i64),
        "sg_host_streamed_count": ([], i64),
        "sg_kernel_info": ([i32, i32, ip, ip, ip, ip, ip, ip, ip, ip], i32),
        "sg_probe_peaks": ([i32, dp, dp, dp], i32),
        "sg_classical": ([i32, vp, vp, vp, i64, i64, i64, vp], i32),
        "sg_classical_block": ([i32, pp, i64, pp, i64, pp, i64, i64, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name, None)
        if fn is None and path != LIB_PATH:
            continue  # an older build under A/B (SG_LIB_PATH)
        if fn is None:
            raise ImportError(f"{path} does not export {name}: rebuild it")
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(rc):
    """Map a status code to the reference's exception types (ValueError for bad input)."""
    if rc == SG_OK:
        return
    msg = load().sg_last_error().decode(errors="replace")
    if rc in (SG_EINVAL, SG_ERANGE, SG_EPATTERN):
        raise ValueError(msg)
    raise SliceGemmError(f"slicegemm_b200 error {rc}: {msg}")


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    return ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)), arr


def current_stream_handle(device=None):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
