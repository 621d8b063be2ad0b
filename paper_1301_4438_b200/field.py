"""Prime-field description shared by the host API (mirror of field.py in the reference).

Restates the modulus validation and storage-dtype rule of
/root/reference/pkg/src/pluq/field.py:19-21, 41-81, 140-147 so that host
matrices carry the same dtype as the reference (float64 for small p, int64
otherwise).  Arithmetic never runs here: device kernels do it.
"""

from __future__ import annotations

from math import isqrt

import numpy as np

DEFAULT_MODULUS_BOUND = 1 << 26
ABSOLUTE_MODULUS_BOUND = 1 << 31

_F64_EXACT = 1 << 53
_I64_EXACT = (1 << 63) - 1


def is_prime(p: int) -> bool:
    """Trial division (field.py:24-38)."""
    if p < 2:
        return False
    if p % 2 == 0:
        return p == 2
    d = 3
    while d <= isqrt(p):
        if p % d == 0:
            return False
        d += 2
    return True


def inverse_mod(a: int, p: int) -> int:
    """Multiplicative inverse mod p; ZeroDivisionError on 0 (field.py:41-52)."""
    a %= p
    if a == 0:
        raise ZeroDivisionError("inverse of 0 requested; upstream pivot logic is broken")
    return pow(a, -1, p)


class PrimeField:
    """Z/pZ with the reference's validation and storage dtype (field.py:55-81)."""

    __slots__ = ("p", "dtype", "max_accumulate", "limbs")

    def __init__(self, p: int, *, allow_large_modulus: bool = False):
        if not isinstance(p, int) or isinstance(p, bool) or not is_prime(p):
            raise ValueError(f"modulus must be a prime integer, got {p!r}")
        bound = ABSOLUTE_MODULUS_BOUND if allow_large_modulus else DEFAULT_MODULUS_BOUND
        if p >= bound:
            raise ValueError(
                f"modulus {p} exceeds the bound {bound}; pass allow_large_modulus=True "
                f"for p up to 2**31 (per-product reduction)"
            )
        self.p = p
        sq = (p - 1) ** 2
        if sq * 8192 <= _F64_EXACT:
            self.dtype = np.float64
            self.max_accumulate = max(1, _F64_EXACT // sq - 1) if sq else _F64_EXACT
        else:
            self.dtype = np.int64
            self.max_accumulate = max(1, _I64_EXACT // sq - 1) if sq else _I64_EXACT
        bits = (p - 1).bit_length()
        self.limbs = max(1, (bits + 7) // 8)  # 8-bit limbs of the tensor-core GEMM

    def __eq__(self, other) -> bool:
        return isinstance(other, PrimeField) and other.p == self.p

    def __hash__(self) -> int:
        return hash(("PrimeField", self.p))

    def __repr__(self) -> str:
        return f"PrimeField({self.p})"

    def add(self, a: int, b: int) -> int:
        return (a + b) % self.p

    def sub(self, a: int, b: int) -> int:
        return (a - b) % self.p

    def neg(self, a: int) -> int:
        return (-a) % self.p

    def mul(self, a: int, b: int) -> int:
        return (a * b) % self.p

    def inv(self, a: int) -> int:
        return inverse_mod(a, self.p)

    def asarray(self, values) -> np.ndarray:
        """Validated canonical residues in the storage dtype (field.py:140-147)."""
        arr = np.asarray(values)
        if arr.size and (np.any(arr < 0) or np.any(arr >= self.p)):
            raise ValueError(f"entries must be canonical residues in [0, {self.p})")
        if arr.dtype != self.dtype:
            arr = arr.astype(self.dtype)
        return arr
