"""Extension fields: ExtFieldSpec, ExtMatrix, ext_multiply (the reference's extension_mul).

Reference contract: SPEC.md:369-431 (extension.py is missing from the reference; names from
__init__.py:17, field objects fields.py:170-219).  A matrix over F_{p^n} is the degree-n
vector of its coefficient matrices over the base field, A = A0 + x A1 (+ x^2 A2).

Two multiplication routes:
  * "karatsuba" -- the reference's algorithm: 3 base-field products for n = 2
    (P0 = A0B0, P2 = A1B1, P1 = (A0+A1)(B0+B1) - P0 - P2) and 6 for n = 3
    (the c0..c4 scheme of SPEC.md:401-406), each an M4RM product on the GPU, then reduction by
    the defining polynomial with add / sub / scalar_mul only.
  * "direct" -- F4 and F8 (characteristic 2): ONE power-basis M4RM product over the 2- / 3-plane
    GF4 / GF8 matrix (fields.GF4, fields.GF8; acc = T[g0] + x T[g1] (+ x^2 T[g2]) with x*
    as a linear map on the planes).  Elements have a unique bit encoding, so the result is
    bit-identical to Karatsuba's.
`ext_multiply` on ExtMatrix operands defaults to "karatsuba", the reference's algorithm, whose
instrumented base-multiply counter reads exactly 3 / 6 per product (acceptance
#4); method="direct" selects the single power-basis product for F4 / F8 (counter 0:
no base-field products; ~25 % faster than three F2 products at 8192^3).  GF4 / GF8
BitslicedMatrix operands -- the power-basis form BASELINE.json's GF(4) config is quoted on --
always take the direct kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .fields import F2, F3, F5, GF4, GF8, FieldSpec
from .m4rm import M4rmParams, m4rm_multiply
from .matrix import BitslicedMatrix


@dataclass(frozen=True)
class ExtFieldSpec:
    """F_p[x] / (modulus); modulus lists coefficients low degree first incl. the leading 1."""

    name: str
    base: FieldSpec
    degree: int
    modulus: tuple
    direct: FieldSpec = None  # power-basis field of the direct kernel (F4, F8)

    def __post_init__(self):
        if self.degree not in (2, 3):
            raise ValueError("only quadratic and cubic extensions supported")
        if len(self.modulus) != self.degree + 1 or self.modulus[-1] != 1:
            raise ValueError("modulus must be monic of the stated degree")
        p = self.base.order
        if any(not 0 <= c < p for c in self.modulus):
            raise ValueError("modulus coefficients must be canonical residues")
        for x in range(p):  # degree 2 or 3: irreducible iff no root
            if sum(c * x ** k for k, c in enumerate(self.modulus)) % p == 0:
                raise ValueError(f"{self.modulus} has root {x} mod {p}: not irreducible")

    @property
    def order(self) -> int:
        return self.base.order ** self.degree

    def __repr__(self):
        return f"ExtFieldSpec({self.name})"


# fields.py:215-219
F4 = ExtFieldSpec("f4", F2, 2, (1, 1, 1), direct=GF4)        # x^2 + x + 1
F8 = ExtFieldSpec("f8", F2, 3, (1, 1, 0, 1), direct=GF8)     # x^3 + x + 1
F9 = ExtFieldSpec("f9", F3, 2, (1, 0, 1))                    # x^2 + 1
F25 = ExtFieldSpec("f25", F5, 2, (3, 0, 1))                  # x^2 - 2
F27 = ExtFieldSpec("f27", F3, 3, (1, 2, 0, 1))               # x^3 - x + 1
EXT_FIELDS = {f.name: f for f in (F4, F8, F9, F25, F27)}

base_multiplies = 0  # base-field products performed by the last ext_multiply


class ExtMatrix:
    """A = A0 + x A1 (+ x^2 A2) with coefficient matrices over spec.base."""

    __slots__ = ("spec", "coeffs")

    def __init__(self, spec: ExtFieldSpec, coeffs):
        if not isinstance(spec, ExtFieldSpec):
            raise TypeError("spec must be an ExtFieldSpec")
        coeffs = list(coeffs)
        if len(coeffs) != spec.degree:
            raise ValueError(f"need {spec.degree} coefficient matrices")
        if any(c.field is not spec.base for c in coeffs):
            raise ValueError(f"coefficient matrices must be over {spec.base.name}")
        shape = (coeffs[0].nrows, coeffs[0].ncols)
        if any((c.nrows, c.ncols) != shape for c in coeffs):
            raise ValueError("coefficient matrices must share a shape")
        self.spec = spec
        self.coeffs = coeffs

    @property
    def nrows(self):
        return self.coeffs[0].nrows

    @property
    def ncols(self):
        return self.coeffs[0].ncols

    @classmethod
    def zero(cls, spec, m, n, device="cuda"):
        return cls(spec, [BitslicedMatrix.zero(spec.base, m, n, device=device) for _ in range(spec.degree)])

    @classmethod
    def from_dense(cls, spec, coeff_dense, device="cuda"):
        """coeff_dense: spec.degree dense residue matrices (low degree first)."""
        return cls(spec, [BitslicedMatrix.from_dense(spec.base, d, device=device) for d in coeff_dense])

    def to_dense(self):
        return [c.to_dense() for c in self.coeffs]

    def as_direct(self) -> BitslicedMatrix:
        """The power-basis matrix (F4 -> GF4, F8 -> GF8): plane i = the F2 coefficient of x^i."""
        if self.spec.direct is None:
            raise ValueError(f"{self.spec.name} has no direct power-basis kernel")
        dev = self.coeffs[0].device
        planes = torch.cat([c.planes.to(dev) for c in self.coeffs], dim=0)
        return BitslicedMatrix(self.spec.direct, self.nrows, self.ncols, planes)

    # backwards-compatible alias
    as_gf4 = as_direct

    @classmethod
    def from_direct(cls, M: BitslicedMatrix) -> "ExtMatrix":
        spec = {GF4: F4, GF8: F8}.get(M.field)
        if spec is None:
            raise ValueError("expected a GF4 or GF8 matrix")
        # plane d of the power-basis matrix is the F2 coefficient matrix of x^d (views, no copy)
        return cls(spec, [BitslicedMatrix(F2, M.nrows, M.ncols, M.planes[d:d + 1])
                          for d in range(spec.degree)])

    from_gf4 = from_direct

    def add(self, other: "ExtMatrix") -> "ExtMatrix":
        _same(self, other)
        return ExtMatrix(self.spec, [a.add(b) for a, b in zip(self.coeffs, other.coeffs)])

    def neg(self) -> "ExtMatrix":
        return ExtMatrix(self.spec, [a.neg() for a in self.coeffs])

    def equals(self, other) -> bool:
        return (isinstance(other, ExtMatrix) and other.spec is self.spec
                and all(a.equals(b) for a, b in zip(self.coeffs, other.coeffs)))


def _same(A, B):
    if A.spec is not B.spec:
        raise ValueError("extension field mismatch")
    if (A.nrows, A.ncols) != (B.nrows, B.ncols):
        raise ValueError("shape mismatch")


def poly_reduce(spec: ExtFieldSpec, P, inplace: bool = False):
    """P0 + x P1 + ... + x^(2n-2) P_(2n-2)  mod  spec.modulus, with add/sub/scalar_mul only
    (SPEC.md:408-413): x^n = -(m_(n-1) x^(n-1) + ... + m_0), applied from the top down.
    inplace: the P_i are temporaries the caller owns (distinct device matrices) and may be
    overwritten -- one launch per subtraction instead of a clone and a launch."""
    n = spec.degree
    P = list(P)
    for top in range(2 * n - 2, n - 1, -1):
        head = P[top]
        for j in range(n):
            c = spec.modulus[j]
            if c:
                t = head.scalar_mul(c) if c != 1 else head
                P[top - n + j] = P[top - n + j]._isub(t) if inplace else P[top - n + j].sub(t)
    return P[:n]


def _sum(x: BitslicedMatrix, y: BitslicedMatrix) -> BitslicedMatrix:
    """x + y of two operand coefficient matrices (not owned: out of place).  Over F2 one XOR kernel."""
    if x.field is F2 and x.device.type == "cuda" and y.device == x.device:
        return BitslicedMatrix(F2, x.nrows, x.ncols, torch.bitwise_xor(x.planes, y.planes))
    return x.add(y)


def _karatsuba(A: ExtMatrix, B: ExtMatrix, params) -> ExtMatrix:
    global base_multiplies
    mul = lambda x, y: m4rm_multiply(x, y, params)  # noqa: E731
    a, b = A.coeffs, B.coeffs
    # the products are fresh matrices owned here: the corrections run in place on them
    if A.spec.degree == 2:
        p0, p2 = mul(a[0], b[0]), mul(a[1], b[1])
        p1 = mul(_sum(a[0], a[1]), _sum(b[0], b[1]))._isub(p0)._isub(p2)
        base_multiplies = 3
        return ExtMatrix(A.spec, poly_reduce(A.spec, [p0, p1, p2], inplace=True))
    c0, c4, m1 = mul(a[0], b[0]), mul(a[2], b[2]), mul(a[1], b[1])
    c1 = mul(_sum(a[0], a[1]), _sum(b[0], b[1]))._isub(c0)._isub(m1)
    c3 = mul(_sum(a[2], a[1]), _sum(b[2], b[1]))._isub(c4)._isub(m1)
    c2 = mul(_sum(a[0], a[2]), _sum(b[0], b[2]))._isub(c0)._isub(c4)._iadd(m1)
    base_multiplies = 6
    # (poly_reduce in place: m1 is not among its inputs, the five c_i are distinct)
    return ExtMatrix(A.spec, poly_reduce(A.spec, [c0, c1, c2, c3, c4], inplace=True))


def ext_multiply(A, B, params: M4rmParams = None, method: str = "karatsuba"):
    """C = A B over an extension field.

    ExtMatrix operands give an ExtMatrix (method "karatsuba" = SPEC.md:393-406, 3 / 6 base
    products; "direct" = one power-basis product for F4 / F8; "auto" = direct where it exists);
    GF4 / GF8 BitslicedMatrix operands (the direct power-basis form) give a BitslicedMatrix of
    the same field."""
    global base_multiplies
    if isinstance(A, BitslicedMatrix) or isinstance(B, BitslicedMatrix):
        if not (isinstance(A, BitslicedMatrix) and isinstance(B, BitslicedMatrix)):
            raise TypeError("mixed ExtMatrix / BitslicedMatrix operands")
        if A.field not in (GF4, GF8) or B.field is not A.field:
            raise ValueError("ext_multiply needs GF4 or GF8 operands of one field")
        base_multiplies = 0
        return m4rm_multiply(A, B, params)
    if not isinstance(A, ExtMatrix) or not isinstance(B, ExtMatrix):
        raise TypeError("ext_multiply takes ExtMatrix operands")
    if A.spec is not B.spec:
        raise ValueError("extension field mismatch")
    if A.ncols != B.nrows:
        raise ValueError(f"inner dimensions {A.ncols} != {B.nrows}")
    if method not in ("auto", "direct", "karatsuba"):
        raise ValueError(f"unknown method {method!r}")
    if method == "direct" or (method == "auto" and A.spec.direct is not None):
        base_multiplies = 0
        return ExtMatrix.from_direct(m4rm_multiply(A.as_direct(), B.as_direct(), params))
    return _karatsuba(A, B, params)
