"""ExtMatrix / ext_multiply for F4 = GF(4) = F2[x]/(x^2+x+1).

Reference contract: SPEC.md:369-431 (extension.py is missing; names from __init__.py:17).  The
reference multiplies F4 matrices by Karatsuba over three F2 products.  This
path multiplies them directly with one 2-plane M4RM over the power basis {1, x}
(acc = T[g0] + x*T[g1], x*(c0, c1) = (c1, c0 ^ c1)): GF(4) elements have a unique 2-bit
encoding, so the result is bit-identical to the Karatsuba result and to oracle_ext_multiply
(oracle.py:192-215).  The coefficient matrices A0 (of 1) and A1 (of x) are exactly the two
planes of the GF4 BitslicedMatrix.
"""

from __future__ import annotations

import torch

from .fields import F2, F4
from .m4rm import M4rmParams, m4rm_multiply
from .matrix import BitslicedMatrix


class ExtMatrix:
    """A = A0 + x*A1 with A0, A1 matrices over F2."""

    __slots__ = ("spec", "coeffs")

    def __init__(self, spec, coeffs):
        if spec is not F4:
            raise ValueError("only F4 = GF(4) is on the B200 path (F8/F9/F25/F27 are listed as next)")
        coeffs = list(coeffs)
        if len(coeffs) != 2 or any(c.field is not F2 for c in coeffs):
            raise ValueError("need 2 coefficient matrices over F2")
        if (coeffs[0].nrows, coeffs[0].ncols) != (coeffs[1].nrows, coeffs[1].ncols):
            raise ValueError("coefficient matrices must share a shape")
        self.spec = spec
        self.coeffs = coeffs

    @property
    def nrows(self):
        return self.coeffs[0].nrows

    @property
    def ncols(self):
        return self.coeffs[0].ncols

    def as_gf4(self) -> BitslicedMatrix:
        c0, c1 = self.coeffs
        dev = c0.device
        planes = torch.cat([c0.planes, c1.planes.to(dev)], dim=0)
        return BitslicedMatrix(F4, self.nrows, self.ncols, planes)

    @classmethod
    def from_gf4(cls, M: BitslicedMatrix) -> "ExtMatrix":
        if M.field is not F4:
            raise ValueError("expected a GF(4) matrix")
        return cls(F4, [BitslicedMatrix(F2, M.nrows, M.ncols, M.planes[d:d + 1].clone()) for d in range(2)])


def ext_multiply(A, B, params: M4rmParams = None):
    """C = A B over GF(4); accepts ExtMatrix or GF4 BitslicedMatrix operands (same type out)."""
    ext = isinstance(A, ExtMatrix)
    a = A.as_gf4() if isinstance(A, ExtMatrix) else A
    b = B.as_gf4() if isinstance(B, ExtMatrix) else B
    if a.field is not F4 or b.field is not F4:
        raise ValueError("ext_multiply needs GF(4) operands")
    C = m4rm_multiply(a, b, params)
    return ExtMatrix.from_gf4(C) if ext else C
