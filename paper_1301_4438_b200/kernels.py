"""Kernel strategy on the GPU: drop-in for ClassicalKernels (/root/reference/pkg/src/pluq/kernels.py:30-120).

``CudaKernels(field)`` exposes the reference's strategy interface
(``mm_acc``, ``trsm_left_unit_lower``, ``trsm_right_upper``) and charges the
same closed-form OpCounts (kernels.py:1-16).  Operands may be CUDA int32 tensor
views (zero-copy) or numpy arrays in the field dtype (copied to the device and
written back in place), so the object can be handed to ``pluq(kernels=...)``
of this package or of the reference itself.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .field import PrimeField
from .matrix import OpCounts


def _torch():
    import torch

    return torch


class _Operand:
    """Device view of an operand (numpy or torch) with write-back for numpy / strided inputs."""

    def __init__(self, x, writable: bool):
        torch = _torch()
        self.src = x
        self.writable = writable
        if isinstance(x, torch.Tensor):
            if not x.is_cuda or x.dtype != torch.int32:
                raise ValueError("device operands must be CUDA int32 tensors")
            if x.ndim == 2 and (x.shape[1] <= 1 or x.stride(1) == 1) and x.stride(0) >= max(1, x.shape[1]):
                self.t = x
                self.copied = False
            else:
                self.t = x.contiguous()
                self.copied = True
        else:
            arr = np.asarray(x)
            dev = torch.device("cuda", torch.cuda.current_device())
            self.t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64)).to(dev).to(torch.int32)
            self.copied = True

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def ld(self) -> int:
        return int(self.t.stride(0)) if self.t.shape[0] > 1 else max(1, int(self.t.shape[1]))

    def finish(self) -> None:
        if not (self.writable and self.copied):
            return
        torch = _torch()
        if isinstance(self.src, torch.Tensor):
            self.src.copy_(self.t)
        else:
            host = self.t.to("cpu").numpy()
            self.src[...] = host.astype(self.src.dtype)


class CudaKernels:
    """B200 kernels behind the reference's strategy interface (kernels.py:30-120)."""

    def __init__(self, field: PrimeField):
        self.field = field

    # -- multiply-accumulate (kernels.py:38-55) --------------------------------------
    def mm_acc(self, c, a, b, counts: OpCounts) -> None:
        m, k = a.shape
        k2, n = b.shape
        if tuple(c.shape) != (m, n) or k2 != k:
            raise ValueError(f"mm_acc shapes C{tuple(c.shape)} A{tuple(a.shape)} B{tuple(b.shape)}")
        if k == 0 or m == 0 or n == 0:
            return
        counts.modular_reductions += m * n
        counts.field_mul += m * n * k
        counts.field_add += m * n * k
        ctx = _native.context()
        oc, oa, ob = _Operand(c, True), _Operand(a, False), _Operand(b, False)
        st = ctx.lib.pluq_modgemm_sub(ctx.handle, oc.ptr, oc.ld, oa.ptr, oa.ld, ob.ptr, ob.ld, m, n, k, self.field.p)
        _native.raise_for(st, ctx, "mm_acc")
        oc.finish()

    # -- triangular solves -----------------------------------------------------------
    def trsm_left_unit_lower(self, l, b, counts: OpCounts) -> None:
        """B <- L^-1 B, L unit lower (kernels.py:59-70)."""
        r = l.shape[0]
        if l.shape[1] != r or b.shape[0] != r:
            raise ValueError(f"trsm shapes L{tuple(l.shape)} B{tuple(b.shape)}")
        n = b.shape[1]
        if r == 0 or n == 0:
            return
        counts.modular_reductions += r * n
        counts.field_mul += n * (r * (r - 1) // 2)
        counts.field_add += n * (r * (r - 1) // 2)
        ctx = _native.context()
        ol, ob = _Operand(l, False), _Operand(b, True)
        st = ctx.lib.pluq_trsm_llu(ctx.handle, ol.ptr, ol.ld, ob.ptr, ob.ld, r, n, self.field.p)
        _native.raise_for(st, ctx, "trsm_left_unit_lower")
        ob.finish()

    def trsm_right_upper(self, b, u, counts: OpCounts) -> None:
        """B <- B U^-1, U upper with nonzero diagonal (kernels.py:85-103)."""
        r = u.shape[0]
        if u.shape[1] != r or b.shape[1] != r:
            raise ValueError(f"trsm shapes B{tuple(b.shape)} U{tuple(u.shape)}")
        m = b.shape[0]
        if r == 0:
            return
        ctx = _native.context()
        ob, ou = _Operand(b, True), _Operand(u, False)
        # the diagonal check happens before any charge (kernels.py:93-96)
        st = ctx.lib.pluq_trsm_ru(ctx.handle, ob.ptr, ob.ld, ou.ptr, ou.ld, 0, r, self.field.p)
        _native.raise_for(st, ctx, "trsm_right_upper")
        counts.field_inv += r
        if m == 0:
            return
        counts.modular_reductions += 2 * m * r
        counts.field_mul += m * (r * (r + 1) // 2)
        counts.field_add += m * (r * (r - 1) // 2)
        st = ctx.lib.pluq_trsm_ru(ctx.handle, ob.ptr, ob.ld, ou.ptr, ou.ld, m, r, self.field.p)
        _native.raise_for(st, ctx, "trsm_right_upper")
        ob.finish()


def device_matmul_mod(x: np.ndarray, y: np.ndarray, p: int) -> np.ndarray:
    """Exact X Y mod p on the device (via C <- 0 - X Y, then negation); int64 result."""
    torch = _torch()
    m, k = x.shape
    n = y.shape[1]
    if m == 0 or n == 0 or k == 0:
        return np.zeros((m, n), dtype=np.int64)
    ctx = _native.context()
    dev = torch.device("cuda", torch.cuda.current_device())
    tx = torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64)).to(dev).to(torch.int32)
    ty = torch.from_numpy(np.ascontiguousarray(y, dtype=np.int64)).to(dev).to(torch.int32)
    tc = torch.zeros((m, n), dtype=torch.int32, device=dev)
    st = ctx.lib.pluq_modgemm_sub(ctx.handle, tc.data_ptr(), n, tx.data_ptr(), k, ty.data_ptr(), n, m, n, k, p)
    _native.raise_for(st, ctx, "matmul_mod")
    out = tc.to("cpu").numpy().astype(np.int64)
    return (p - out) % p


# The reference exports its kernel strategy as ``ClassicalKernels`` (pluq/__init__.py:11,49;
# kernels.py:30-120); user code written against it (``pluq.ClassicalKernels(field)``) gets the
# CUDA strategy, which has the same interface and charges.
ClassicalKernels = CudaKernels
