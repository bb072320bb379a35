"""paper_0901_1413_b200: the bitsliced Method-of-Four-Russians product over F3, F5, F7 and
GF(4) (with F2, Z/4, Z/8, GF(8) and, by Karatsuba, F9 / F25 / F27), B200-native.

A drop-in for the multiply path of the reference package `slicegemm` (arXiv:0901.1413,
Boothby & Bradshaw): the same matrix type, packing and multiply API (slicegemm/__init__.py:15-17,
SPEC.md:198-431) over hand-written sm_100a kernels in libslicegemm_b200.so, called through the
C ABI in include/slicegemm_b200.h.  There is no CPU fallback.
"""

from .fields import F2, F3, F5, F7, GF4, GF8, Z4, Z8, FIELDS, BasisElement, FieldSpec, by_name
from .matrix import BitslicedMatrix, RowRef, row_accumulate
from .dense import DenseMatrix
from .m4rm import M4rmParams, build_table, choose_k, classical_multiply, m4rm_multiply, plan
from .extension import EXT_FIELDS, F4, F8, F9, F25, F27, ExtFieldSpec, ExtMatrix, ext_multiply, poly_reduce
from . import _core_cuda

__version__ = "0.1.0"


def backend_name() -> str:
    """Name of the active backend (slicegemm.backend_name, __init__.py:13)."""
    return _core_cuda.NAME


__all__ = [
    "BitslicedMatrix", "DenseMatrix", "RowRef", "row_accumulate", "ExtFieldSpec", "ExtMatrix", "M4rmParams", "FieldSpec",
    "F2", "F3", "F4", "F5", "F7", "F8", "F9", "F25", "F27", "GF4", "GF8", "Z4", "Z8", "FIELDS", "EXT_FIELDS",
    "backend_name", "build_table", "by_name", "choose_k", "classical_multiply", "ext_multiply", "m4rm_multiply", "plan", "poly_reduce",
]
