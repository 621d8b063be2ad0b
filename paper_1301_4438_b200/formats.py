"""Text formats of matrices and factorizations.

Same files as the reference (`/root/reference/pkg/src/pluq/matrix.py:128-158` for a
matrix, `:351-375` for a factorization), so files written by either package load in the
other:

* matrix: a header line ``m n p`` then m lines of n residues separated by spaces;
* factors: ``m n p r``, the m entries of P.sigma, the n entries of Q.sigma, then the
  packed matrix in the matrix format.

Parsing raises ``ValueError`` on the reference's error cases (empty file, malformed header,
negative dimensions, wrong row count or width, trailing non-blank lines, entries outside
[0, p) — the last through the ``DenseMatrix`` constructor).  Device-resident matrices are
copied to the host for writing.
"""

from __future__ import annotations

import numpy as np


def matrix_to_text(a) -> str:
    data = a.host_array()
    out = [f"{a.m} {a.n} {a.p}"]
    out.extend(" ".join(map(str, row)) for row in data.tolist())
    return "\n".join(out) + "\n"


def matrix_from_text(text: str):
    from .field import PrimeField
    from .matrix import DenseMatrix

    lines = text.splitlines()
    if not lines or not lines[0].strip():
        raise ValueError("empty matrix file")
    head = lines[0].split()
    if len(head) != 3:
        raise ValueError(f"bad matrix header {lines[0]!r}, expected 'm n p'")
    m, n, p = (int(v) for v in head)
    if m < 0 or n < 0:
        raise ValueError("negative dimensions")
    field = PrimeField(p)
    rows = lines[1:1 + m]
    if len(rows) != m or any(extra.strip() for extra in lines[1 + m:]):
        raise ValueError(f"expected exactly {m} rows after the header")
    data = np.zeros((m, n), dtype=np.int64)
    for i, line in enumerate(rows):
        vals = line.split()
        if len(vals) != n:
            raise ValueError(f"row {i} has {len(vals)} entries, expected {n}")
        if n:
            data[i] = np.array([int(v) for v in vals], dtype=np.int64)
    return DenseMatrix(field, data)


def factors_to_text(f) -> str:
    head = f"{f.m} {f.n} {f.packed.p} {f.rank}"
    return "\n".join([head, f.p_perm.serialize(), f.q_perm.serialize(), matrix_to_text(f.packed)])


def factors_from_text(text: str):
    from .matrix import Permutation, PluqFactors

    lines = text.splitlines()
    if len(lines) < 4:
        raise ValueError("truncated factor file")
    head = lines[0].split()
    if len(head) != 4:
        raise ValueError(f"bad factor header {lines[0]!r}, expected 'm n p r'")
    m, n, p, r = (int(v) for v in head)
    P = Permutation.deserialize(lines[1], size=m)
    Q = Permutation.deserialize(lines[2], size=n)
    packed = matrix_from_text("\n".join(lines[3:]))
    if packed.shape != (m, n) or packed.p != p:
        raise ValueError("factor header disagrees with the packed matrix header")
    if not 0 <= r <= min(m, n):
        raise ValueError(f"rank {r} out of range")
    return PluqFactors(P, Q, r, packed)
