"""Field descriptors for the B200 path (a restatement of the reference's FieldSpec data).

Names, orders and encodings follow slicegemm/fields.py: F2 (:78-86), F3 unit/sign planes
(:88-101), F5 and F7 plain 3-bit redundant patterns (:103-129), the rings Z4 / Z8 (:131-158).
GF4 / GF8 are GF(4) = F2[x]/(x^2+x+1) and GF(8) = F2[x]/(x^3+x+1) (:215-216) stored directly as
2- / 3-plane matrices whose plane i is the coefficient of x^i (an element's residue code r in
[0, q) is the polynomial sum_i ((r >> i) & 1) x^i).  The reference's extension-field objects
(F4, F8, F9, F25, F27 as ExtFieldSpec) live in extension.py.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib


@dataclass(frozen=True)
class BasisElement:
    """One additive-basis component alpha and how its 0/1 coefficient is read off a pattern:
    ("plane", d) = bit d, ("xor", d, e) = bit d XOR bit e (fields.py:16-32).  The M4RM index of
    the basis element for a row is exactly this extraction applied to A's planes (_core_py.py:
    186-202)."""

    alpha: int
    extract: tuple

    def coefficient(self, pattern: int) -> int:
        kind = self.extract[0]
        bit = (pattern >> self.extract[1]) & 1
        return bit ^ ((pattern >> self.extract[2]) & 1) if kind == "xor" else bit


def _binary_basis(planes: int) -> tuple:
    return tuple(BasisElement(1 << d, ("plane", d)) for d in range(planes))


@dataclass(frozen=True)
class FieldSpec:
    name: str
    order: int
    char: int
    bits: int               # bit planes per element
    code: int               # SG_* field code of the C ABI
    decode_table: tuple     # pattern -> residue (None = illegal)
    canonical_table: tuple  # residue -> pattern
    basis: tuple = ()       # BasisElement per lookup (the kernels' index planes)
    is_field: bool = True

    @property
    def valid_patterns(self) -> frozenset:
        return frozenset(i for i, r in enumerate(self.decode_table) if r is not None)

    def decode(self, pattern: int) -> int:
        e = self.decode_table[pattern]
        if e is None:
            raise ValueError(f"invalid {self.name} pattern {pattern:#b}")
        return e

    def canonical(self, residue: int) -> int:
        if not 0 <= residue < self.order:
            raise ValueError(f"{residue} is not a residue of {self.name}")
        return self.canonical_table[residue]

    def basis_coefficients(self, pattern: int) -> tuple:
        return tuple(b.coefficient(pattern) for b in self.basis)

    def __repr__(self):
        return f"FieldSpec({self.name})"


F2 = FieldSpec("f2", 2, 2, 1, _lib.SG_F2, (0, 1), (0, 1), _binary_basis(1))
# F3: unit / sign planes; basis {1, -1}: the "+1" coefficient is unit XOR sign, "-1" the sign
F3 = FieldSpec("f3", 3, 3, 2, _lib.SG_F3, (0, 1, None, 2), (0, 1, 3),
               (BasisElement(1, ("xor", 0, 1)), BasisElement(2, ("plane", 1))))
F5 = FieldSpec("f5", 5, 5, 3, _lib.SG_F5, (0, 1, 2, 3, 4, 0, 1, 2), (0, 1, 2, 3, 4), _binary_basis(3))
F7 = FieldSpec("f7", 7, 7, 3, _lib.SG_F7, (0, 1, 2, 3, 4, 5, 6, 0), (0, 1, 2, 3, 4, 5, 6), _binary_basis(3))
Z4 = FieldSpec("z4", 4, 4, 2, _lib.SG_Z4, (0, 1, 2, 3), (0, 1, 2, 3), _binary_basis(2), is_field=False)
Z8 = FieldSpec("z8", 8, 8, 3, _lib.SG_Z8, tuple(range(8)), tuple(range(8)), _binary_basis(3), is_field=False)
# GF(4) / GF(8) power-basis matrices: residue code r <-> polynomial sum ((r >> i) & 1) x^i; the
# basis is {1, x (, x^2)}, alpha = the residue code of x^i.
GF4 = FieldSpec("gf4", 4, 2, 2, _lib.SG_GF4, (0, 1, 2, 3), (0, 1, 2, 3), _binary_basis(2))
GF8 = FieldSpec("gf8", 8, 2, 3, _lib.SG_GF8, tuple(range(8)), tuple(range(8)), _binary_basis(3))

FIELDS = {f.name: f for f in (F2, F3, F5, F7, Z4, Z8)}
ALL_FIELDS = {**FIELDS, "gf4": GF4, "gf8": GF8, "f4": GF4, "f8": GF8}


def by_name(name: str) -> FieldSpec:
    try:
        return ALL_FIELDS[name.lower()]
    except KeyError:
        raise ValueError(f"unknown field {name!r}") from None
