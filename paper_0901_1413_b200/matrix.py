"""BitslicedMatrix: the reference's matrix type, stored plane-major in B200 HBM.

Contract: SPEC.md:198-299 (the reference's matrix.py is missing, __init__.py:15).  Storage is
one int64 tensor of shape (R, nrows, words_per_row) holding the exact uint64 bit patterns of
the reference layout: plane d holds bit d of every entry, column c -> word c >> 6, bit c & 63,
padding lanes zero.  A matrix may live on a CUDA device (where
every operation runs, through libslicegemm_b200.so) or on the host as a plain container; a
host matrix is moved to the GPU by any operation that computes, and m4rm_multiply on two host
matrices runs the host-buffer entry point sg_m4rm_host (copies included).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .fields import FieldSpec, by_name


def _words(n: int) -> int:
    return (n + 63) // 64


def _dev(device):
    d = torch.device(device)
    if d.type == "cuda" and d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return d


class one_cpu_writer:
    """Context: the calling thread on the CPU it is running on and torch's CPU ops single-threaded
    (both restored on exit) -- host buffers written inside are written by one thread on one CPU."""

    def __enter__(self):
        self.threads = torch.get_num_threads()
        self.mask = None
        try:
            cpu = ctypes.CDLL(None).sched_getcpu()
            if cpu >= 0 and hasattr(__import__("os"), "sched_setaffinity"):
                import os
                self.mask = os.sched_getaffinity(0)
                os.sched_setaffinity(0, {cpu})
        except (OSError, AttributeError):
            self.mask = None
        torch.set_num_threads(1)
        return self

    def __exit__(self, *exc):
        torch.set_num_threads(self.threads)
        if self.mask is not None:
            import os
            os.sched_setaffinity(0, self.mask)
        return False


def _require_cuda(device):
    if device.type != "cuda":
        raise ValueError("this operation runs on a CUDA device (no CPU fallback)")
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device is available: the B200 path has no CPU fallback")


def _vp(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


class BitslicedMatrix:
    __slots__ = ("field", "nrows", "ncols", "planes")

    def __init__(self, field: FieldSpec, nrows: int, ncols: int, planes: torch.Tensor):
        if isinstance(field, str):
            field = by_name(field)
        if nrows < 0 or ncols < 0:
            raise ValueError("dimensions must be non-negative")
        shape = (field.bits, nrows, _words(ncols))
        if tuple(planes.shape) != shape or planes.dtype != torch.int64:
            raise ValueError(f"planes must be int64 of shape {shape}, got {tuple(planes.shape)} {planes.dtype}")
        self.field = field
        self.nrows = nrows
        self.ncols = ncols
        self.planes = planes.contiguous()

    # ------------------------------------------------------------------ construction
    @property
    def words_per_row(self) -> int:
        return _words(self.ncols)

    @property
    def device(self) -> torch.device:
        return self.planes.device

    @classmethod
    def zero(cls, field, m: int, n: int, device="cuda") -> "BitslicedMatrix":
        if isinstance(field, str):
            field = by_name(field)
        if m < 0 or n < 0:
            raise ValueError("dimensions must be non-negative")
        return cls(field, m, n, torch.zeros((field.bits, m, _words(n)), dtype=torch.int64, device=device))

    @classmethod
    def from_planes(cls, field, planes, n: int, device=None) -> "BitslicedMatrix":
        """Wrap reference-layout planes (numpy uint64 (R, m, W) or a torch int64 tensor)."""
        if isinstance(field, str):
            field = by_name(field)
        if isinstance(planes, np.ndarray):
            t = torch.from_numpy(np.ascontiguousarray(planes, dtype=np.uint64).view(np.int64))
        else:
            t = planes
        if device is not None:
            t = t.to(device)
        return cls(field, t.shape[1], n, t)

    @classmethod
    def from_dense(cls, field, D, device="cuda") -> "BitslicedMatrix":
        """Pack dense residues (numpy / torch / an object with .entries) on the GPU."""
        if isinstance(field, str):
            field = by_name(field)
        entries = getattr(D, "entries", D)
        if isinstance(entries, torch.Tensor):
            if entries.dtype.is_floating_point:
                raise ValueError("entries must be integers")
            if entries.dtype != torch.uint8 and entries.numel() and (
                    int(entries.min()) < 0 or int(entries.max()) >= field.order):
                raise ValueError(f"entries out of range for {field.name}")
            dense = entries.to(torch.uint8)
        else:
            arr = np.asarray(entries)
            if arr.ndim != 2:
                raise ValueError("entries must be two-dimensional")
            if not np.issubdtype(arr.dtype, np.integer):
                raise ValueError("entries must be integers")
            # wider integer types must be checked before the uint8 cast (256 would wrap to 0);
            # uint8 entries are range-checked by the pack kernel itself
            if arr.dtype != np.uint8 and arr.size and (arr.min() < 0 or arr.max() >= field.order):
                raise ValueError(f"entries out of range for {field.name}")
            dense = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.uint8))
        if dense.dim() != 2:
            raise ValueError("entries must be two-dimensional")
        m, n = dense.shape
        target = _dev(device)
        gpu = target if target.type == "cuda" else _dev("cuda")
        _require_cuda(gpu)
        if m and n:  # the pack kernel writes every plane word (padding lanes as zeros): no zero fill first
            out = cls(field, m, n, torch.empty((field.bits, m, _words(n)), dtype=torch.int64, device=gpu))
        else:
            out = cls.zero(field, m, n, device=gpu)
        if m and n:
            dd = dense.to(gpu, non_blocking=False).contiguous()
            with torch.cuda.device(gpu):
                st = _lib.current_stream_handle(gpu)
                L = _lib.load()
                _lib.check(L.sg_pack(field.code, _vp(dd), m, n, n, _vp(out.planes), st))
                _lib.check(L.sg_stream_check(st))  # ValueError on an entry that is not a residue
        return out if target.type == "cuda" else out.to(target)

    @classmethod
    def random(cls, field, m: int, n: int, seed: int, device="cuda") -> "BitslicedMatrix":
        """Deterministic uniform residues: the DenseMatrix.random stream (oracle.py:47-50)."""
        if isinstance(field, str):
            field = by_name(field)
        from .dense import DenseMatrix
        dense = np.asarray(DenseMatrix.random(field, m, n, seed))
        return cls.from_dense(field, dense, device=device)

    # ------------------------------------------------------------------ movement
    def to(self, device) -> "BitslicedMatrix":
        return BitslicedMatrix(self.field, self.nrows, self.ncols, self.planes.to(device))

    def cpu(self) -> "BitslicedMatrix":
        return self.to("cpu")

    def cuda(self, device=None) -> "BitslicedMatrix":
        return self.to(_dev("cuda" if device is None else device))

    def copy(self) -> "BitslicedMatrix":
        return BitslicedMatrix(self.field, self.nrows, self.ncols, self.planes.clone())

    def pin_memory(self) -> "BitslicedMatrix":
        """A copy in page-locked host memory, the operand form of the host-buffer path (copied
        asynchronously, overlapped with the products).  The buffer is allocated and filled by
        the calling thread alone, kept on one CPU while it does: on the B200 box (a 16-vCPU VM)
        host-to-device DMA from page-locked buffers written by several threads at once ran at
        15-25 GB/s instead of ~52 in most processes (profiles/r02_experiments.txt)."""
        with one_cpu_writer():
            t = torch.empty(tuple(self.planes.shape), dtype=torch.int64, pin_memory=True)
            t.copy_(self.planes)
        return BitslicedMatrix(self.field, self.nrows, self.ncols, t)

    @classmethod
    def pinned_zero(cls, field, m: int, n: int) -> "BitslicedMatrix":
        """An all-zero page-locked host matrix (an `out` for the host-buffer path), written as
        pin_memory's buffers are."""
        if isinstance(field, str):
            field = by_name(field)
        with one_cpu_writer():
            t = torch.zeros((field.bits, m, _words(n)), dtype=torch.int64, pin_memory=True)
        return cls(field, m, n, t)

    @classmethod
    def pinned_empty(cls, field, m: int, n: int) -> "BitslicedMatrix":
        """An uninitialized page-locked host matrix: the result buffer of a host-buffer product,
        every word of which (padding lanes included) is copied down from the device."""
        if isinstance(field, str):
            field = by_name(field)
        return cls(field, m, n, torch.empty((field.bits, m, _words(n)), dtype=torch.int64, pin_memory=True))

    def planes_numpy(self) -> np.ndarray:
        """The reference-layout planes as a host uint64 array of shape (R, m, W)."""
        return self.planes.cpu().numpy().view(np.uint64)

    def _on_gpu(self) -> "BitslicedMatrix":
        return self if self.device.type == "cuda" else self.cuda()

    # ------------------------------------------------------------------ dense views
    def to_dense(self) -> "DenseMatrix":
        """Unpack to a DenseMatrix: residues unpacked on the GPU, returned on the host.

        The result behaves like the reference's DenseMatrix (.field, .nrows, .ncols, .entries as
        an int64 (m, n) array, ==) and converts to a numpy array with np.asarray (uint8)."""
        from .dense import DenseMatrix
        return DenseMatrix._trusted(self.field, self.to_numpy())

    def to_numpy(self) -> np.ndarray:
        """Unpack to dense residues (uint8, shape (m, n)) on the GPU, returned on the host."""
        g = self._on_gpu()
        _require_cuda(g.device)
        out = torch.empty((self.nrows, self.ncols), dtype=torch.uint8, device=g.device)
        if self.nrows and self.ncols:
            with torch.cuda.device(g.device):
                st = _lib.current_stream_handle(g.device)
                L = _lib.load()
                _lib.check(L.sg_unpack(self.field.code, _vp(g.planes), self.nrows, self.ncols, _vp(out),
                                       self.ncols, st))
                _lib.check(L.sg_stream_check(st))  # ValueError on an illegal F3 pattern
        return out.cpu().numpy()

    def get(self, i: int, j: int) -> int:
        if not (0 <= i < self.nrows and 0 <= j < self.ncols):
            raise IndexError("index out of range")
        words = self.planes[:, i, j >> 6].cpu().numpy().view(np.uint64)
        pat = sum(int((int(words[d]) >> (j & 63)) & 1) << d for d in range(self.field.bits))
        return self.field.decode(pat)

    def set(self, i: int, j: int, e: int) -> None:
        if not (0 <= i < self.nrows and 0 <= j < self.ncols):
            raise IndexError("index out of range")
        pat = self.field.canonical(e)
        words = self.planes[:, i, j >> 6].cpu().numpy().view(np.uint64).copy()
        bit = np.uint64(1 << (j & 63))
        for d in range(self.field.bits):
            if (pat >> d) & 1:
                words[d] |= bit
            else:
                words[d] &= ~bit
        self.planes[:, i, j >> 6] = torch.from_numpy(words.view(np.int64)).to(self.device)

    # ------------------------------------------------------------------ elementwise (GPU)
    def _check_same(self, other: "BitslicedMatrix"):
        if not isinstance(other, BitslicedMatrix) or other.field is not self.field:
            raise ValueError("field mismatch")
        if (other.nrows, other.ncols) != (self.nrows, self.ncols):
            raise ValueError("shape mismatch")

    def _plane_op(self, op: str, src: "BitslicedMatrix" = None, scalar: int = 0, tail=True):
        dst = self._on_gpu().copy()
        R = self.field.bits
        dptr, _k1 = _lib.ptr_array([dst.planes[d].data_ptr() for d in range(R)])
        if src is not None:
            s = src.planes.to(dst.device).contiguous()
            sptr, _k2 = _lib.ptr_array([s[d].data_ptr() for d in range(R)])
        else:
            sptr = None
        rem = self.ncols % 64
        tmask = ((1 << rem) - 1) if (rem and tail) else (1 << 64) - 1
        if self.nrows and self.words_per_row:
            with torch.cuda.device(dst.device):
                _lib.check(_lib.load().sg_plane_op(_lib.OPS[op], dptr, sptr, self.nrows, self.words_per_row,
                                                   tmask, scalar, _lib.current_stream_handle(dst.device)))
        return dst

    def _iplane_op(self, op: str, src: "BitslicedMatrix" = None, scalar: int = 0) -> "BitslicedMatrix":
        """`_plane_op` in place on a device matrix the caller owns (a temporary of a longer
        computation: no clone, one launch); host matrices take the out-of-place route."""
        if self.device.type != "cuda" or not self.planes.is_contiguous():
            return self._plane_op(op, src, scalar)
        R = self.field.bits
        dptr, _k1 = _lib.ptr_array([self.planes[d].data_ptr() for d in range(R)])
        sptr = None
        if src is not None:
            s = src.planes.to(self.device).contiguous()
            sptr, _k2 = _lib.ptr_array([s[d].data_ptr() for d in range(R)])
        rem = self.ncols % 64
        tmask = ((1 << rem) - 1) if rem else (1 << 64) - 1
        if self.nrows and self.words_per_row:
            with torch.cuda.device(self.device):
                _lib.check(_lib.load().sg_plane_op(_lib.OPS[op], dptr, sptr, self.nrows, self.words_per_row,
                                                   tmask, scalar, _lib.current_stream_handle(self.device)))
        return self

    def _isub(self, other: "BitslicedMatrix") -> "BitslicedMatrix":
        self._check_same(other)
        return self._iplane_op(self._SUB[self.field.name], other)

    def _iadd(self, other: "BitslicedMatrix") -> "BitslicedMatrix":
        self._check_same(other)
        return self._iplane_op(self._ADD[self.field.name], other)

    _ADD = {"f2": "f2_add", "f3": "f3_add", "f5": "f5_add", "f7": "f7_add", "gf4": "gf4_add", "gf8": "gf8_add",
            "z4": "z4_add", "z8": "z8_add"}
    _SUB = {"f2": "f2_add", "f3": "f3_sub", "f5": "f5_sub", "f7": "f7_sub", "gf4": "gf4_add", "gf8": "gf8_add",
            "z4": "z4_sub", "z8": "z8_sub"}
    _NEG = {"f3": "f3_neg", "f5": "f5_neg", "f7": "f7_neg", "z4": "z4_neg", "z8": "z8_neg"}
    _SMUL = {"f3": "scalar_mul_f3", "f5": "scalar_mul_f5", "f7": "scalar_mul_f7", "gf4": "scalar_mul_gf4",
             "gf8": "scalar_mul_gf8", "z4": "scalar_mul_z4", "z8": "scalar_mul_z8"}

    def add(self, other: "BitslicedMatrix") -> "BitslicedMatrix":
        self._check_same(other)
        return self._plane_op(self._ADD[self.field.name], other)

    def sub(self, other: "BitslicedMatrix") -> "BitslicedMatrix":
        self._check_same(other)
        return self._plane_op(self._SUB[self.field.name], other)

    def neg(self) -> "BitslicedMatrix":
        name = self.field.name
        if name not in self._NEG:  # characteristic 2: -x = x
            return self._on_gpu().copy()
        return self._plane_op(self._NEG[name])

    def scalar_mul(self, c: int) -> "BitslicedMatrix":
        if not 0 <= c < self.field.order:
            raise ValueError(f"{c} is not a residue of {self.field.name}")
        name = self.field.name
        if name == "f2":
            return self._on_gpu().copy() if c else BitslicedMatrix.zero(self.field, self.nrows, self.ncols,
                                                                       self._on_gpu().device)
        return self._plane_op(self._SMUL[name], scalar=c)

    def reduce_canonical(self) -> "BitslicedMatrix":
        out = self._on_gpu().copy()
        if self.nrows and self.ncols:
            with torch.cuda.device(out.device):
                _lib.check(_lib.load().sg_reduce_canonical(self.field.code, _vp(out.planes), self.nrows,
                                                           self.ncols, _lib.current_stream_handle(out.device)))
        return out

    def equals(self, other) -> bool:
        """True iff the decoded entries agree (canonicalizes internally)."""
        if not isinstance(other, BitslicedMatrix) or other.field is not self.field:
            return False
        if (other.nrows, other.ncols) != (self.nrows, self.ncols):
            return False
        a = self.reduce_canonical().planes
        b = other.reduce_canonical().planes.to(a.device)
        return bool(torch.equal(a, b))

    __eq__ = equals
    __hash__ = None

    def row(self, i: int) -> "RowRef":
        """A view of row i across every plane."""
        return RowRef(self, i)

    def __repr__(self):
        return f"BitslicedMatrix({self.field.name}, {self.nrows}x{self.ncols}, {self.device})"


class RowRef:
    """One row of a BitslicedMatrix across all R planes: R word slices of words_per_row words
    (SPEC.md:210-213).  A view -- row_accumulate on it updates the parent matrix in place."""

    __slots__ = ("matrix", "index")

    def __init__(self, matrix: BitslicedMatrix, index: int):
        if not isinstance(matrix, BitslicedMatrix):
            raise TypeError("RowRef needs a BitslicedMatrix")
        if not 0 <= index < matrix.nrows:
            raise IndexError(f"row {index} out of range for {matrix.nrows} rows")
        self.matrix = matrix
        self.index = index

    @property
    def field(self) -> FieldSpec:
        return self.matrix.field

    @property
    def ncols(self) -> int:
        return self.matrix.ncols

    @property
    def words(self) -> torch.Tensor:
        """The (R, words_per_row) int64 view of the row's plane words."""
        return self.matrix.planes[:, self.index]

    def to_list(self) -> list:
        return [self.matrix.get(self.index, j) for j in range(self.ncols)]

    def __repr__(self):
        return f"RowRef({self.field.name}, row {self.index} of {self.matrix.nrows}x{self.ncols})"


_ROW_OPS = {("f2", "add"): "f2_add", ("f2", "sub"): "f2_add", ("f3", "add"): "f3_add", ("f3", "sub"): "f3_sub",
            ("f5", "add"): "f5_add", ("f5", "sub"): "f5_sub", ("f7", "add"): "f7_add", ("f7", "sub"): "f7_sub",
            ("z4", "add"): "z4_add", ("z4", "sub"): "z4_sub", ("z8", "add"): "z8_add", ("z8", "sub"): "z8_sub",
            ("gf4", "add"): "gf4_add", ("gf4", "sub"): "gf4_add", ("gf8", "add"): "gf8_add",
            ("gf8", "sub"): "gf8_add"}


def row_accumulate(dst: RowRef, src: RowRef, mode: str = "add") -> None:
    """dst <- dst +/- src lanewise through the field's plane kernel, in place.

    The row's words are updated on the GPU (one sg_plane_op launch over one row); a row of a
    host matrix is moved to the GPU and back.  Padding lanes stay zero (F7 sub re-masks them).
    Errors: field or length mismatch (ValueError), unknown mode."""
    if not isinstance(dst, RowRef) or not isinstance(src, RowRef):
        raise TypeError("row_accumulate takes two RowRef")
    if dst.field is not src.field:
        raise ValueError(f"field mismatch: {dst.field.name} vs {src.field.name}")
    if dst.ncols != src.ncols:
        raise ValueError(f"row lengths differ: {dst.ncols} vs {src.ncols}")
    if mode not in ("add", "sub"):
        raise ValueError(f"mode must be 'add' or 'sub', not {mode!r}")
    f = dst.field
    W = dst.matrix.words_per_row
    if W == 0:
        return
    M = dst.matrix
    dev = M.device if M.device.type == "cuda" else _dev("cuda")
    _require_cuda(dev)
    on_dev = M.device.type == "cuda"
    # (R, W): a strided view into the device matrix (updated in place), or a device copy of a host row
    d = M.planes[:, dst.index] if on_dev else M.planes[:, dst.index].to(dev).contiguous()
    s = src.matrix.planes[:, src.index].to(dev)
    R = f.bits
    # each plane's row is a contiguous run of W words; its pointer is the view's row d
    stride = d.stride(0) * 8
    dptr, _k1 = _lib.ptr_array([d.data_ptr() + p * stride for p in range(R)])
    sptr, _k2 = _lib.ptr_array([s.data_ptr() + p * s.stride(0) * 8 for p in range(R)])
    rem = M.ncols % 64
    tail = ((1 << rem) - 1) if rem else (1 << 64) - 1
    with torch.cuda.device(dev):
        _lib.check(_lib.load().sg_plane_op(_lib.OPS[_ROW_OPS[(f.name, mode)]], dptr, sptr, 1, W, tail, 0,
                                           _lib.current_stream_handle(dev)))
    if not on_dev:
        M.planes[:, dst.index] = d.cpu()
