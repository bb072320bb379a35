"""DenseMatrix: the reference's row-major matrix of canonical residues (oracle.py:17-66).

`BitslicedMatrix.to_dense()` returns one, and `BitslicedMatrix.from_dense` accepts
one, so a caller written against the reference's `DenseMatrix` (field, entries, nrows, ncols,
zero / identity / random, copy, equals / ==) runs unchanged.  Entries are held as the uint8
residues the unpack kernel produced; `.entries` is the reference's int64 view (made on first
use), and `np.asarray(D)` gives the uint8 array without a copy, so large unpacked matrices do
not pay for an 8-byte-per-entry conversion unless the caller asks for it.
"""

from __future__ import annotations

import numpy as np

from .fields import FieldSpec, by_name


class DenseMatrix:
    __slots__ = ("field", "_u8", "_i64")

    def __init__(self, field, entries):
        if isinstance(field, str):
            field = by_name(field)
        arr = np.asarray(entries)
        if arr.ndim != 2:
            raise ValueError("entries must be two-dimensional")
        if arr.dtype != np.uint8 or not arr.flags.c_contiguous:
            if arr.size and not np.issubdtype(arr.dtype, np.integer):
                arr = np.array(entries, dtype=np.int64)
            if arr.size and (arr.min() < 0 or arr.max() >= field.order):
                raise ValueError(f"entries out of range for {field.name}")
            arr = np.ascontiguousarray(arr, dtype=np.uint8)
        elif arr.size and arr.max() >= field.order:
            raise ValueError(f"entries out of range for {field.name}")
        self.field = field
        self._u8 = arr
        self._i64 = None

    @classmethod
    def _trusted(cls, field: FieldSpec, u8: np.ndarray) -> "DenseMatrix":
        """Wrap residues the unpack kernel produced (already canonical and in range)."""
        d = cls.__new__(cls)
        d.field, d._u8, d._i64 = field, u8, None
        return d

    # ---------------------------------------------------------------- reference API
    @property
    def entries(self) -> np.ndarray:
        if self._i64 is None:
            self._i64 = self._u8.astype(np.int64)
        return self._i64

    @property
    def nrows(self) -> int:
        return self._u8.shape[0]

    @property
    def ncols(self) -> int:
        return self._u8.shape[1]

    @classmethod
    def zero(cls, field, m: int, n: int) -> "DenseMatrix":
        return cls(field, np.zeros((m, n), dtype=np.uint8))

    @classmethod
    def identity(cls, field, n: int) -> "DenseMatrix":
        return cls(field, np.eye(n, dtype=np.uint8))

    @classmethod
    def random(cls, field, m: int, n: int, seed: int) -> "DenseMatrix":
        """The reference's seeded draw (oracle.py:47-50): PCG64(seed).integers(0, order, (m, n),
        int64), drawn in row chunks (the same stream as one monolithic draw)."""
        if isinstance(field, str):
            field = by_name(field)
        g = np.random.Generator(np.random.PCG64(seed))
        out = np.empty((m, n), dtype=np.uint8)
        step = max(1, (1 << 24) // max(n, 1))
        for r0 in range(0, m, step):
            r1 = min(m, r0 + step)
            out[r0:r1] = g.integers(0, field.order, size=(r1 - r0, n), dtype=np.int64)
        return cls._trusted(field, out)

    def copy(self) -> "DenseMatrix":
        return DenseMatrix._trusted(self.field, self._u8.copy())

    def equals(self, other) -> bool:
        return (isinstance(other, DenseMatrix) and self.field is other.field
                and self._u8.shape == other._u8.shape and bool(np.array_equal(self._u8, other._u8)))

    def __eq__(self, other):
        if isinstance(other, DenseMatrix):
            return self.equals(other)
        return NotImplemented

    __hash__ = None

    def __repr__(self):
        return f"DenseMatrix({self.field.name}, {self.nrows}x{self.ncols})"

    # ---------------------------------------------------------------- array interop
    def __array__(self, dtype=None, copy=None):
        return self._u8 if dtype is None else self._u8.astype(dtype)

    @property
    def shape(self) -> tuple:
        return self._u8.shape

    def astype(self, dtype) -> np.ndarray:
        return self._u8.astype(dtype)

    def __getitem__(self, idx):
        return self._u8[idx]

    def __len__(self) -> int:
        return self._u8.shape[0]
