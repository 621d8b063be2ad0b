"""Device-side verification of a factorization.

``freivalds(original, factors)`` checks Mat(P) [L;M] [U V] Mat(Q) == A (mod p)
with random probe vectors: A x == P (L (U (Q x))) costs O((m+n) r) per probe on the
device instead of the O(m n r) dense reconstruction, so it scales to the full
BASELINE configs where the CPU oracle cannot run.  Also checks the packed
structure (nonzero U diagonal, zero trailing block) on the device.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .matrix import DenseMatrix, PluqFactors


def _mm(a, b, p):
    """C = A B mod p for CUDA int32 tensors via the native modular GEMM (C <- 0 - A B)."""
    import torch

    m, k = a.shape
    n = b.shape[1]
    c = torch.zeros((m, n), dtype=torch.int32, device=a.device)
    if m == 0 or n == 0 or k == 0:
        return c
    a = a.contiguous()
    b = b.contiguous()
    ctx = _native.context(a.device.index)
    st = ctx.lib.pluq_modgemm_sub(ctx.handle, c.data_ptr(), n, a.data_ptr(), k, b.data_ptr(), n, m, n, k, p)
    _native.raise_for(st, ctx, "freivalds gemm")
    c.neg_().add_(p)  # c = -AB mod p  ->  AB mod p, in place
    return c.masked_fill_(c == p, 0)


def freivalds(original, factors: PluqFactors, probes: int = 4, seed: int = 0) -> bool:
    """True iff the factorization reproduces ``original`` on `probes` random probe blocks."""
    import torch

    p = factors.packed.p
    packed = factors.packed.data if factors.packed.on_device else factors.packed.to_device().data
    dev = packed.device
    a = original.data if isinstance(original, DenseMatrix) else original
    if not isinstance(a, torch.Tensor):
        a = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int64))).to(dev).to(torch.int32)
    m, n = packed.shape
    r = factors.rank
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randint(0, p, (n, probes), generator=g, dtype=torch.int64).to(dev).to(torch.int32)
    lhs = _mm(a, x, p)
    # Q x : Mat(Q) has 1 at (t, sigma(t)), so (Q x)[t] = x[sigma(t)]
    qs = torch.from_numpy(factors.q_perm.sigma).to(dev)
    y = x[qs]
    uv = packed[:r, :].clone()
    if r:
        uv[:, :r] = torch.triu(uv[:, :r])
    z = _mm(uv, y, p)                       # r x probes
    lm = torch.tril(packed[:, :r], -1).clone()
    if r:
        lm[torch.arange(r, device=dev), torch.arange(r, device=dev)] = 1
    w = _mm(lm, z, p)                       # m x probes
    ps = torch.from_numpy(factors.p_perm.sigma).to(dev)
    rhs = w[ps]                              # (Mat(P) w)[i] = w[sigma(i)]
    return bool(torch.equal(lhs, rhs))


def structure_ok(factors: PluqFactors) -> bool:
    """Device version of PluqFactors.check_structure (matrix.py:337-349)."""
    import torch

    packed = factors.packed.data if factors.packed.on_device else factors.packed.to_device().data
    r = factors.rank
    if r:
        d = torch.diagonal(packed[:r, :r])
        if bool((d == 0).any()):
            return False
    return not bool((packed[r:, r:] != 0).any())
