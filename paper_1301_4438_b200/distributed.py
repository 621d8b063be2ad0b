"""One large matrix across ranks: block-column distributed generic-profile LU.

SURVEY §8(e) / BASELINE north star: for a single large matrix the trailing
Schur-complement update is partitioned across GPUs and the pivot panels are broadcast
(NCCL over NVLink on the GPU box, gloo in the CPU tests); the recursion and the base case
stay on one GPU.

Layout: column panels of width W, panel k (columns [kW, kW+W)) owned by rank k % N for
all m rows (a 1 x N process grid of the 2D block partition).  Step k:
  1. the owner factors the panel below row kW on its GPU with the exact single-GPU path
     (`pluq_factor`, speculative generic LU inside);
  2. the panel is broadcast; every rank turns the pivot rows of its later panels into U
     (L11^-1 A12, TRSM) and updates the rows below (A22 -= L21 U12, tensor-core GEMM).
The generic-profile facts used by the single-GPU path (tests/test_generic_profile.py)
make the assembled result exactly the reference's: A is generic iff every panel is
generic after the preceding updates; then P = Q = I, the packed output is the unique LU
and OpCounts depend on (m, n, r, threshold) only.  A rank-deficient panel (zero pivot at
g) ends the factorization if the whole Schur complement vanishes (all-reduce); any
non-generic panel makes rank 0 run the exact single-GPU `pluq` on the original matrix,
which is only overwritten by the final gather.

Kernels go through a backend object (`CudaPanelBackend` in the product: C ABI on this
rank's GPU); there is no CPU fallback in the product path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .field import PrimeField
from .matrix import DenseMatrix, OpCounts, Permutation, PluqFactors

DEFAULT_PANEL = 1024


class CudaPanelBackend:
    """Panel operations on CUDA int32 tensors through the C ABI (this rank's device)."""

    def __init__(self, p: int, threshold: int, device: int):
        self.p, self.threshold, self.device = int(p), int(threshold), device
        self.ctx = _native.context(device)
        self.lib = self.ctx.lib

    def factor_panel(self, x):
        """In-place exact PLUQ of a contiguous panel; returns (rank, generic)."""
        m, n = x.shape
        P = np.empty(m, np.int64)
        Q = np.empty(n, np.int64)
        r = np.zeros(1, np.int64)
        c = np.zeros(4, np.int64)
        st = self.lib.pluq_factor(self.ctx.handle, x.data_ptr(), x.stride(0), m, n, self.p, self.threshold,
                                  _native.i64p(P), _native.i64p(Q), _native.i64p(r), _native.i64p(c))
        _native.raise_for(st, self.ctx, "pluq_factor (panel)")
        generic = bool(np.array_equal(P, np.arange(m)) and np.array_equal(Q, np.arange(n)))
        return int(r[0]), generic

    def trsm_llu(self, l, b):
        """b <- l^-1 b, l unit lower (strided views)."""
        st = self.lib.pluq_trsm_llu(self.ctx.handle, l.data_ptr(), l.stride(0), b.data_ptr(), b.stride(0),
                                    l.shape[0], b.shape[1], self.p)
        _native.raise_for(st, self.ctx, "pluq_trsm_llu")

    def gemm_sub(self, c, a, b):
        """c <- c - a b mod p (strided views)."""
        st = self.lib.pluq_modgemm_sub(self.ctx.handle, c.data_ptr(), c.stride(0), a.data_ptr(), a.stride(0),
                                       b.data_ptr(), b.stride(0), c.shape[0], c.shape[1], a.shape[1], self.p)
        _native.raise_for(st, self.ctx, "pluq_modgemm_sub")

    def is_zero(self, x) -> bool:
        out = ctypes.c_int64(0)
        st = self.lib.pluq_nonzero(self.ctx.handle, x.data_ptr(), x.stride(0), x.shape[0], x.shape[1],
                                   ctypes.byref(out))
        _native.raise_for(st, self.ctx, "pluq_nonzero")
        return out.value == 0


def panel_bounds(n: int, width: int) -> list[tuple[int, int]]:
    return [(c0, min(c0 + width, n)) for c0 in range(0, n, width)]


def panel_owner(k: int, world: int) -> int:
    return k % world


def _world():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


class LocalSlab:
    """The panels a rank owns, side by side in ONE m x (sum of widths) tensor, so that its
    later panels are always a contiguous column range (one TRSM + one GEMM per step)."""

    def __init__(self, tensor, owned, offsets, widths):
        self.t, self.owned, self.off, self.w = tensor, owned, offsets, widths

    def panel(self, k):
        return self.t[:, self.off[k]:self.off[k] + self.w[k]]

    def after(self, k):
        """Columns of the owned panels j > k (a contiguous view, possibly empty)."""
        later = [j for j in self.owned if j > k]
        if not later:
            return None
        return self.t[:, self.off[later[0]]:]


def _layout(n: int, width: int, rank: int, world: int):
    owned, offsets, widths, col = [], {}, {}, 0
    for k, (c0, c1) in enumerate(panel_bounds(n, width)):
        if panel_owner(k, world) == rank:
            owned.append(k)
            offsets[k], widths[k] = col, c1 - c0
            col += c1 - c0
    return owned, offsets, widths, col


def scatter_panels(a_full, m: int, n: int, width: int, make_empty) -> LocalSlab:
    """Rank 0 holds a_full (m x n); every rank receives the panels it owns."""
    import torch.distributed as dist

    rank, world = _world()
    owned, offsets, widths, cols = _layout(n, width, rank, world)
    slab = LocalSlab(make_empty(m, cols), owned, offsets, widths)
    for k, (c0, c1) in enumerate(panel_bounds(n, width)):
        owner = panel_owner(k, world)
        if owner == 0 and rank == 0:
            slab.panel(k).copy_(a_full[:, c0:c1])
        elif rank == 0:
            dist.send(a_full[:, c0:c1].contiguous(), dst=owner)
        elif rank == owner:
            buf = make_empty(m, c1 - c0)
            dist.recv(buf, src=0)
            slab.panel(k).copy_(buf)
    return slab


def gather_panels(slab: LocalSlab, a_full, m: int, n: int, width: int, make_empty):
    """Inverse of scatter_panels: rank 0 writes every panel back into a_full."""
    import torch.distributed as dist

    rank, world = _world()
    for k, (c0, c1) in enumerate(panel_bounds(n, width)):
        owner = panel_owner(k, world)
        if owner == 0 and rank == 0:
            a_full[:, c0:c1] = slab.panel(k)
        elif rank == 0:
            buf = make_empty(m, c1 - c0)
            dist.recv(buf, src=owner)
            a_full[:, c0:c1] = buf
        elif rank == owner:
            dist.send(slab.panel(k).contiguous(), dst=0)


def distributed_generic_lu(slab: LocalSlab, m: int, n: int, width: int, backend, flags):
    """Factor the distributed panels in place.  Returns the rank r when the matrix has a
    generic rank profile (then P = Q = I), or None when it does not (panels are then
    partially updated; the caller restarts from the original on one GPU)."""
    import torch.distributed as dist

    rank, world = _world()
    mn = min(m, n)
    for k, (c0, c1) in enumerate(panel_bounds(n, width)):
        if c0 >= mn:
            break
        owner = panel_owner(k, world)
        wk = c1 - c0
        flag = flags()
        pan = flags.new_panel(m - c0, wk)  # contiguous broadcast buffer
        if rank == owner:
            pview = slab.panel(k)[c0:, :]
            rk, generic = backend.factor_panel(pview)
            pan.copy_(pview)
            flag[0], flag[1] = rk, int(generic)
        if world > 1:
            dist.broadcast(flag, src=owner)
        rk, generic = int(flag[0]), bool(int(flag[1]))
        if not generic:
            return None
        if world > 1:
            dist.broadcast(pan, src=owner)
        g = c0 + rk
        rest = slab.after(k)
        if rest is not None and rk > 0:
            top = rest[c0:g, :]
            backend.trsm_llu(pan[:rk, :rk], top)                  # U12: pivot rows of the later panels
            if g < m:
                backend.gemm_sub(rest[g:, :], pan[rk:, :rk], top)  # A22 -= L21 U12
        if rk < wk:
            # zero pivot at g: generic only if the whole Schur complement A[g:, g:] vanishes
            # (panel k's own part was checked by the exact panel factorization)
            nz = flags()
            nz[0] = int(rest is not None and g < m and not backend.is_zero(rest[g:, :]))
            if world > 1:
                dist.all_reduce(nz, op=dist.ReduceOp.MAX)
            return g if int(nz[0]) == 0 else None
    return mn


class _Flags:
    """Small int64 flag tensors and panel receive buffers on the backend's device."""

    def __init__(self, device, dtype):
        import torch

        self.torch, self.device, self.dtype = torch, device, dtype

    def __call__(self):
        return self.torch.zeros(2, dtype=self.torch.int64, device=self.device)

    def new_panel(self, rows, cols):
        return self.torch.empty((rows, cols), dtype=self.dtype, device=self.device)

    def empty(self, rows, cols):
        return self.new_panel(rows, cols)


def pluq_distributed(a: DenseMatrix | None, m: int, n: int, p: int, threshold: int = 30,
                     width: int = DEFAULT_PANEL, counts: OpCounts | None = None, backend=None,
                     device=None):
    """pluq() of one large matrix held by rank 0 (CUDA int32 DenseMatrix), with the
    trailing updates spread over every rank of the default process group.  All ranks call
    it; rank 0 gets the PluqFactors (in place, `f.packed is a`), the others get the rank."""
    import torch

    rank, world = _world()
    if threshold < 1:
        raise ValueError("threshold must be a positive integer")
    field = PrimeField(p)
    if device is None:
        device = a.data.device if (rank == 0 and a is not None) else torch.device("cuda", torch.cuda.current_device())
    if backend is None:
        backend = CudaPanelBackend(p, threshold, device.index if device.type == "cuda" else 0)
    flags = _Flags(device, torch.int32 if device.type == "cuda" else torch.int64)
    if rank == 0:
        x = a.data
        if tuple(x.shape) != (m, n):
            raise ValueError("shape mismatch")
        full = x.clone()  # the original stays untouched until the final gather
    else:
        full = None
    slab = scatter_panels(full, m, n, width, flags.empty)
    r = distributed_generic_lu(slab, m, n, width, backend, flags)
    if r is not None:
        gather_panels(slab, full if rank == 0 else None, m, n, width, flags.empty)
    if rank != 0:
        return r
    if r is None:  # not generic: the exact recursion on one GPU, from the untouched original
        from .recursive import pluq

        return pluq(a, threshold=threshold, counts=counts)
    a.data.copy_(full)
    if counts is not None:
        c = np.zeros(4, np.int64)
        _native.raise_for(_native.load_library().pluq_generic_counts(m, n, r, threshold, _native.i64p(c)), None,
                          "pluq_generic_counts")
        counts.field_mul += int(c[0]); counts.field_add += int(c[1])
        counts.field_inv += int(c[2]); counts.modular_reductions += int(c[3])
    return PluqFactors(Permutation(np.arange(m, dtype=np.int64)), Permutation(np.arange(n, dtype=np.int64)), r, a)
