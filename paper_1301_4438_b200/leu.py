"""PLUQ -> LEU conversion (reference leu.py:79-105).

From the factors of ``pluq()`` (Z-curve pivoting),

    Lbar = P [L 0; M I] P^T,   E = P [I_r; 0] Q,   Ubar = Q^T [U V; 0 0] Q

give A = Lbar E Ubar with Lbar unit lower and Ubar upper triangular.  As in the reference
the triangularity (a property of the pivot order, not of PLUQ in general) and the product
identity are CHECKED, not trusted: ``to_leu`` raises ``RuntimeError`` if either fails.

Device-first: for a device-resident factorization the dense m x m / n x n factors are built
on the GPU by index scatters and the product check runs on the package's modular GEMM
(Lbar E is a column gather, so only one GEMM); host factorizations use numpy.  The dense
LEU is O(m^2 + n^2) memory — the reference notes it is impractical at scale, so use it at
sizes where that fits.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .matrix import DenseMatrix, PluqFactors


@dataclass
class LeuFactors:
    lbar: DenseMatrix  # m x m unit lower triangular
    e: DenseMatrix     # m x n, r ones in distinct rows and columns
    ubar: DenseMatrix  # n x n upper triangular

    @property
    def p(self) -> int:
        return self.lbar.p


def _lower_upper_dense(f: PluqFactors, y, z, xp):
    """P [L 0; M Y] P^T and Q^T [U V; 0 Z] Q with the array module xp (numpy or torch)."""
    m, n, r = f.m, f.n, f.rank
    lm, uv = f.extract_lm(), f.extract_uv()
    if xp is np:
        low = np.zeros((m, m), dtype=np.int64)
        up = np.zeros((n, n), dtype=np.int64)
        low[:, :r] = lm
        low[r:, r:] = y
        up[:r, :] = uv
        up[r:, r:] = z
        sp, qi = f.p_perm.sigma, f.q_perm.inverse().sigma
        return low[np.ix_(sp, sp)], up[np.ix_(qi, qi)]
    torch = xp
    dev = lm.device
    low = torch.zeros((m, m), dtype=torch.int32, device=dev)
    up = torch.zeros((n, n), dtype=torch.int32, device=dev)
    low[:, :r] = lm
    low[r:, r:] = y
    up[:r, :] = uv
    up[r:, r:] = z
    sp = torch.from_numpy(f.p_perm.sigma).to(dev)
    qi = torch.from_numpy(f.q_perm.inverse().sigma).to(dev)
    return low[sp][:, sp], up[qi][:, qi]


def check_triangular_extension(factors: PluqFactors, y, z) -> tuple[bool, bool]:
    """Whether P[L 0; M Y]P^T is unit lower and Q^T[U V; 0 Z]Q upper triangular (leu.py:57-76)."""
    m, n, r = factors.m, factors.n, factors.rank
    if tuple(y.shape) != (m - r, m - r):
        raise ValueError(f"Y must be {(m - r, m - r)}, got {tuple(y.shape)}")
    if tuple(z.shape) != (n - r, n - r):
        raise ValueError(f"Z must be {(n - r, n - r)}, got {tuple(z.shape)}")
    if factors.packed.on_device:
        import torch

        dev = factors.packed.data.device
        lo, up = _lower_upper_dense(factors, torch.as_tensor(np.asarray(y), dtype=torch.int32, device=dev),
                                    torch.as_tensor(np.asarray(z), dtype=torch.int32, device=dev), torch)
        ones = bool((torch.diagonal(lo) == 1).all())
        return (ones and not bool(torch.triu(lo, 1).any())), not bool(torch.tril(up, -1).any())
    lo, up = _lower_upper_dense(factors, np.asarray(y), np.asarray(z), np)
    return (bool(np.all(np.triu(lo, 1) == 0) and np.all(np.diagonal(lo) == 1)), bool(np.all(np.tril(up, -1) == 0)))


def to_leu(factors: PluqFactors, original: DenseMatrix) -> LeuFactors:
    """Dense LEU factors, verified against ``original`` (leu.py:79-105)."""
    field = factors.packed.field
    m, n, r = factors.m, factors.n, factors.rank
    if original.shape != (m, n) or original.p != field.p:
        raise ValueError("original matrix does not match the factors")
    pairs = factors.support_pairs()
    rows = np.array([a for a, _ in pairs], dtype=np.int64)
    cols = np.array([b for _, b in pairs], dtype=np.int64)
    if factors.packed.on_device:
        import torch

        from .verify import _mm

        dev = factors.packed.data.device
        lbar, ubar = _lower_upper_dense(factors, torch.eye(m - r, dtype=torch.int32, device=dev),
                                        torch.zeros((n - r, n - r), dtype=torch.int32, device=dev), torch)
        e = torch.zeros((m, n), dtype=torch.int32, device=dev)
        if r:
            e[torch.from_numpy(rows).to(dev), torch.from_numpy(cols).to(dev)] = 1
        if not (bool((torch.diagonal(lbar) == 1).all()) and not bool(torch.triu(lbar, 1).any())):
            raise RuntimeError("LEU integrity failure: Lbar is not unit lower triangular")
        if bool(torch.tril(ubar, -1).any()):
            raise RuntimeError("LEU integrity failure: Ubar is not upper triangular")
        # Lbar E keeps column a_t of Lbar in column b_t: a gather, then one modular GEMM
        le = torch.zeros((m, n), dtype=torch.int32, device=dev)
        if r:
            le[:, torch.from_numpy(cols).to(dev)] = lbar[:, torch.from_numpy(rows).to(dev)]
        prod = _mm(le, ubar.contiguous(), field.p)
        orig = original.data if original.on_device else torch.from_numpy(original.host_array()).to(dev).to(torch.int32)
        if not torch.equal(prod, orig):
            raise RuntimeError("LEU integrity failure: Lbar E Ubar != A")
        return LeuFactors(DenseMatrix(field, lbar.contiguous()), DenseMatrix(field, e), DenseMatrix(field, ubar.contiguous()))
    lbar, ubar = _lower_upper_dense(factors, np.eye(m - r, dtype=np.int64), np.zeros((n - r, n - r), np.int64), np)
    e = np.zeros((m, n), dtype=np.int64)
    e[rows, cols] = 1
    if not (np.all(np.triu(lbar, 1) == 0) and np.all(np.diagonal(lbar) == 1)):
        raise RuntimeError("LEU integrity failure: Lbar is not unit lower triangular")
    if not np.all(np.tril(ubar, -1) == 0):
        raise RuntimeError("LEU integrity failure: Ubar is not upper triangular")
    from .kernels import device_matmul_mod

    le = np.zeros((m, n), dtype=np.int64)
    le[:, cols] = lbar[:, rows]
    prod = np.asarray(device_matmul_mod(le, ubar, field.p), dtype=np.int64)
    if not np.array_equal(prod, original.host_array()):
        raise RuntimeError("LEU integrity failure: Lbar E Ubar != A")
    return LeuFactors(DenseMatrix(field, lbar), DenseMatrix(field, e), DenseMatrix(field, ubar))
