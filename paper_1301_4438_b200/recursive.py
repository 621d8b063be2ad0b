"""Public PLUQ entry points (mirror of /root/reference/pkg/src/pluq/recursive.py, iterative.py).

``pluq(a, threshold=30, counts=None, kernels=None, workspace=None)`` keeps the
reference signature and contract (recursive.py:159-183): ``a`` is consumed in
place (``f.packed is a``), P/Q are fresh ``Permutation`` objects, OpCounts are
charged exactly as the reference charges them.

* ``kernels is None and workspace is None`` (the default): the whole recursion
  runs in the native driver (libpluq_b200.so) on device-resident data.
* otherwise the recursion is driven from Python over CUDA tensor views, calling
  the injected strategy object (``CudaKernels`` or a subclass) for every
  mm_acc / trsm and the workspace for every auxiliary buffer — the reference's
  two injection points, kept for instrumentation.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .field import PrimeField
from .kernels import CudaKernels
from .matrix import DenseMatrix, OpCounts, Permutation, PluqFactors, apply_cols, apply_rows, perm_block_diag

DEFAULT_THRESHOLD = 30


def _torch_dtype(dtype):
    """torch dtype of a Workspace request: torch dtypes as given, numpy dtypes mapped, and
    None -> int32 (device residues are int32 whatever the host field dtype)."""
    import torch

    if dtype is None:
        return torch.int32
    if isinstance(dtype, torch.dtype):
        return dtype
    return torch.from_numpy(np.zeros(0, dtype=np.dtype(dtype))).dtype


class Workspace:
    """Source of auxiliary element buffers (recursive.py:36-48); device tensors here."""

    def element_buffer(self, shape, dtype=None):
        import torch

        shape = (shape,) if isinstance(shape, int) else tuple(shape)
        return torch.zeros(shape, dtype=_torch_dtype(dtype), device=torch.device("cuda", torch.cuda.current_device()))

    def release(self, buf) -> None:
        pass


class TrackingWorkspace(Workspace):
    """Workspace recording live/peak element counts (recursive.py:51-74)."""

    def __init__(self):
        self.live_elements = 0
        self.peak_elements = 0
        self.scratch_blocks: list[int] = []
        self._sizes: dict[int, int] = {}

    def element_buffer(self, shape, dtype=None):
        buf = super().element_buffer(shape, dtype)
        self._sizes[id(buf)] = buf.numel()
        self.live_elements += buf.numel()
        self.peak_elements = max(self.peak_elements, self.live_elements)
        if buf.ndim == 2:
            self.scratch_blocks.append(buf.numel())
        return buf

    def release(self, buf) -> None:
        self.live_elements -= self._sizes.pop(id(buf), 0)

    @property
    def max_scratch_block(self) -> int:
        return max(self.scratch_blocks, default=0)


def build_s_perm(r1: int, r2: int, r3: int, r4: int, k: int, m: int) -> Permutation:
    """Row block permutation S (recursive.py:77-85)."""
    if not (0 <= r1 + r2 <= k <= m and 0 <= r3 + r4 <= m - k):
        raise ValueError(f"inconsistent row block sizes ({r1},{r2},{r3},{r4},k={k},m={m})")
    a, c = r1 + r2, r3 + r4
    sigma = np.arange(m, dtype=np.int64)
    sigma[a:k] = np.arange(a, k) + c
    sigma[k:k + c] = np.arange(k, k + c) - (k - a)
    return Permutation(sigma)


def build_t_perm(r1: int, r2: int, r3: int, r4: int, k: int, n: int) -> Permutation:
    """Column block permutation T (recursive.py:88-99): sigma[j] = source column of slot j."""
    if not (0 <= r1 + r3 <= k <= n and 0 <= r2 + r4 <= n - k):
        raise ValueError(f"inconsistent column block sizes ({r1},{r2},{r3},{r4},k={k},n={n})")
    blocks = [(0, r1), (k, r2), (r1, r3), (k + r2, r4), (r1 + r3, k - r1 - r3), (k + r2 + r4, n - k - r2 - r4)]
    sigma = np.concatenate([np.arange(s, s + w, dtype=np.int64) for s, w in blocks])
    return Permutation(sigma)


# ------------------------------------------------------------------------------------
# native entry points
# ------------------------------------------------------------------------------------


def _native_factor(a: DenseMatrix, threshold: int, counts: OpCounts, iterative: bool):
    m, n = a.shape
    if m == 0 or n == 0:  # (recursive.py:188-189): nothing to factor, no device work
        return Permutation.identity(m), Permutation.identity(n), 0
    psig = np.zeros(m, dtype=np.int64)
    qsig = np.zeros(n, dtype=np.int64)
    rank = np.zeros(1, dtype=np.int64)
    cnt = np.zeros(4, dtype=np.int64)
    ctx = _native.context(a.data.device.index if a.on_device else None)
    lib = ctx.lib
    if a.on_device:
        x = a.data
        if x.shape[1] > 1 and x.stride(1) != 1:
            raise ValueError("device matrix must be row-major")
        ld = int(x.stride(0)) if m > 1 else max(n, 1)
        if iterative:
            st = lib.pluq_factor_iterative(ctx.handle, x.data_ptr(), ld, m, n, a.p, _native.i64p(psig),
                                           _native.i64p(qsig), _native.i64p(rank), _native.i64p(cnt))
        else:
            st = lib.pluq_factor(ctx.handle, x.data_ptr(), ld, m, n, a.p, threshold, _native.i64p(psig),
                                 _native.i64p(qsig), _native.i64p(rank), _native.i64p(cnt))
        _native.raise_for(st, ctx, "pluq")
    else:
        if iterative:
            # Alg. 2 on the host buffer: stage through the device
            dev = a.to_device()
            f = _native_factor(dev, threshold, counts, True)
            a.data[...] = dev.data.to("cpu").numpy().astype(a.data.dtype)
            return f
        arr = a.data
        work = arr if arr.flags.c_contiguous else np.ascontiguousarray(arr)
        fn = lib.pluq_factor_host_f64 if work.dtype == np.float64 else lib.pluq_factor_host_i64
        if work.dtype not in (np.float64, np.int64):
            raise ValueError(f"host matrices must be float64 or int64, got {work.dtype}")
        st = fn(ctx.handle, work.ctypes.data, m, n, a.p, threshold, _native.i64p(psig), _native.i64p(qsig),
                _native.i64p(rank), _native.i64p(cnt))
        _native.raise_for(st, ctx, "pluq")
        if work is not arr:
            arr[...] = work
    counts.add_array(cnt)
    return Permutation(psig), Permutation(qsig), int(rank[0])


def last_stats() -> dict:
    """Driver statistics of the last native factorization on this thread's context."""
    return _native.context().stats()


# ------------------------------------------------------------------------------------
# instrumented driver (strategy / workspace injection), Algorithm 1 over device views
# ------------------------------------------------------------------------------------


def _base_dev(x, p: int, counts: OpCounts):
    """Alg. 2 on a device view via the native base case (iterative.py:30-93)."""
    m, n = x.shape
    if m == 0 or n == 0:
        return Permutation.identity(m), Permutation.identity(n), 0
    psig = np.zeros(m, dtype=np.int64)
    qsig = np.zeros(n, dtype=np.int64)
    rank = np.zeros(1, dtype=np.int64)
    cnt = np.zeros(4, dtype=np.int64)
    ctx = _native.context(x.device.index)
    ld = int(x.stride(0)) if m > 1 else max(n, 1)
    st = ctx.lib.pluq_factor_iterative(ctx.handle, x.data_ptr(), ld, m, n, p, _native.i64p(psig),
                                       _native.i64p(qsig), _native.i64p(rank), _native.i64p(cnt))
    _native.raise_for(st, ctx, "base case")
    counts.add_array(cnt)
    return Permutation(psig), Permutation(qsig), int(rank[0])


def _rec_dev(x, p, threshold, counts, kernels, ws):
    m, n = x.shape
    ident = Permutation.identity
    if m == 0 or n == 0:
        return ident(m), ident(n), 0
    if m == 1 or n == 1 or min(m, n) <= threshold:
        return _base_dev(x, p, counts)
    kr, kc = m // 2, n // 2
    p1, q1, r1 = _rec_dev(x[:kr, :kc], p, threshold, counts, kernels, ws)
    apply_rows(x[:kr, kc:], p1.inverse())
    apply_cols(x[kr:, :kc], q1.inverse())
    kernels.trsm_left_unit_lower(x[:r1, :r1], x[:r1, kc:], counts)
    kernels.trsm_right_upper(x[kr:, :r1], x[:r1, :r1], counts)
    kernels.mm_acc(x[r1:kr, kc:], x[r1:kr, :r1], x[:r1, kc:], counts)
    kernels.mm_acc(x[kr:, r1:kc], x[kr:, :r1], x[:r1, r1:kc], counts)
    kernels.mm_acc(x[kr:, kc:], x[kr:, :r1], x[:r1, kc:], counts)
    p2, q2, r2 = _rec_dev(x[r1:kr, kc:], p, threshold, counts, kernels, ws)
    p3, q3, r3 = _rec_dev(x[kr:, r1:kc], p, threshold, counts, kernels, ws)
    apply_rows(x[kr:, kc:], p3.inverse())
    apply_cols(x[kr:, kc:], q2.inverse())
    apply_rows(x[kr:, :r1], p3.inverse())
    apply_rows(x[r1:kr, :r1], p2.inverse())
    apply_cols(x[:r1, kc:], q2.inverse())
    apply_cols(x[:r1, r1:kc], q3.inverse())
    u2 = x[r1:r1 + r2, kc:kc + r2]
    l3 = x[kr:kr + r3, r1:r1 + r3]
    kernels.trsm_right_upper(x[kr:kr + r3, kc:kc + r2], u2, counts)
    scratch = ws.element_buffer((r3, r2), x.dtype)
    scratch.copy_(x[kr:kr + r3, kc:kc + r2])
    kernels.trsm_left_unit_lower(l3, scratch, counts)
    kernels.trsm_right_upper(x[kr + r3:, kc:kc + r2], u2, counts)
    kernels.trsm_left_unit_lower(l3, x[kr:kr + r3, kc + r2:], counts)
    kernels.mm_acc(x[kr:kr + r3, kc + r2:], scratch, x[r1:r1 + r2, kc + r2:], counts)
    ws.release(scratch)
    kernels.mm_acc(x[kr + r3:, kc + r2:], x[kr + r3:, kc:kc + r2], x[r1:r1 + r2, kc + r2:], counts)
    kernels.mm_acc(x[kr + r3:, kc + r2:], x[kr + r3:, r1:r1 + r3], x[kr:kr + r3, kc + r2:], counts)
    p4, q4, r4 = _rec_dev(x[kr + r3:, kc + r2:], p, threshold, counts, kernels, ws)
    apply_rows(x[kr + r3:, :kc + r2], p4.inverse())
    apply_cols(x[:kr + r3, kc + r2:], q4.inverse())
    s_perm = build_s_perm(r1, r2, r3, r4, kr, m)
    t_perm = build_t_perm(r1, r2, r3, r4, kc, n)
    apply_rows(x, s_perm.inverse())
    apply_cols(x, t_perm.inverse())
    p_left = p1.compose(perm_block_diag([ident(r1), p2]))
    p_right = p3.compose(perm_block_diag([ident(r3), p4]))
    p_perm = perm_block_diag([p_left, p_right]).compose(s_perm)
    q_left = perm_block_diag([ident(r1), q3]).compose(q1)
    q_right = perm_block_diag([ident(r2), q4]).compose(q2)
    q_perm = t_perm.compose(perm_block_diag([q_left, q_right]))
    return p_perm, q_perm, r1 + r2 + r3 + r4


# ------------------------------------------------------------------------------------
# public API
# ------------------------------------------------------------------------------------


def pluq(
    a: DenseMatrix,
    threshold: int = DEFAULT_THRESHOLD,
    counts: OpCounts | None = None,
    kernels=None,
    workspace: Workspace | None = None,
) -> PluqFactors:
    """PLUQ of ``a`` in place; returns PluqFactors sharing ``a`` (recursive.py:159-183)."""
    if threshold < 1:
        raise ValueError("threshold must be a positive integer")
    counts = counts if counts is not None else OpCounts()
    if kernels is None and workspace is None:
        p_perm, q_perm, rank = _native_factor(a, threshold, counts, iterative=False)
        return PluqFactors(p_perm, q_perm, rank, a)
    kernels = kernels if kernels is not None else CudaKernels(a.field)
    ws = workspace if workspace is not None else Workspace()
    dev = a if a.on_device else a.to_device()
    rowbuf = ws.element_buffer(a.n, dev.data.dtype)
    colbuf = ws.element_buffer(a.m, dev.data.dtype)
    try:
        p_perm, q_perm, rank = _rec_dev(dev.data, a.p, threshold, counts, kernels, ws)
    finally:
        ws.release(rowbuf)
        ws.release(colbuf)
    if not a.on_device:
        a.data[...] = dev.data.to("cpu").numpy().astype(a.data.dtype)
    return PluqFactors(p_perm, q_perm, rank, a)


def pluq_iterative(a: DenseMatrix, counts: OpCounts | None = None) -> PluqFactors:
    """Algorithm 2 on the whole matrix, in place (iterative.py:23-27)."""
    counts = counts if counts is not None else OpCounts()
    p_perm, q_perm, rank = _native_factor(a, 1, counts, iterative=True)
    return PluqFactors(p_perm, q_perm, rank, a)


def base_case_row(a: DenseMatrix, counts: OpCounts | None = None) -> PluqFactors:
    """1 x n case (recursive.py:112-116); bit-identical to Alg. 2 on a row."""
    if a.m != 1:
        raise ValueError("base_case_row needs a single row")
    return pluq_iterative(a, counts)


def base_case_col(a: DenseMatrix, counts: OpCounts | None = None) -> PluqFactors:
    """m x 1 case (recursive.py:119-123); bit-identical to Alg. 2 on a column."""
    if a.n != 1:
        raise ValueError("base_case_col needs a single column")
    return pluq_iterative(a, counts)


class BatchedPluq:
    """Result of ``pluq_batched``: stacked sigmas, ranks and the packed batch (in place)."""

    def __init__(self, field, packed, p_sigma, q_sigma, ranks, counts=None):
        self.field = field
        self.packed = packed
        self.p_sigma = p_sigma
        self.q_sigma = q_sigma
        self.ranks = ranks
        self.counts = counts

    def __len__(self):
        return int(self.ranks.shape[0])

    def factors(self, b: int) -> PluqFactors:
        """PluqFactors view of matrix ``b`` (packed copied to host)."""
        import torch

        blk = self.packed[b]
        host = blk.to("cpu").numpy().astype(np.int64) if isinstance(blk, torch.Tensor) else np.asarray(blk, np.int64)
        ps = self.p_sigma[b]
        qs = self.q_sigma[b]
        ps = ps.to("cpu").numpy() if isinstance(ps, torch.Tensor) else ps
        qs = qs.to("cpu").numpy() if isinstance(qs, torch.Tensor) else qs
        return PluqFactors(Permutation(ps), Permutation(qs), int(self.ranks[b]), DenseMatrix(self.field, host))


def pluq_batched(data, p: int, threshold: int = DEFAULT_THRESHOLD, with_counts: bool = False) -> BatchedPluq:
    """PLUQ of every matrix of a (B, m, n) batch, in place — one CTA per matrix.

    ``data``: CUDA int32 tensor (device-resident; outputs stay on device) or a
    numpy float64 array (host buffers; the call copies in and out).  Each matrix
    gets exactly the factors ``pluq(DenseMatrix(..), threshold)`` would produce.
    """
    import torch

    if threshold < 1:
        raise ValueError("threshold must be a positive integer")
    field = PrimeField(p)
    if isinstance(data, torch.Tensor):
        if data.ndim != 3 or not data.is_cuda or data.dtype != torch.int32 or not data.is_contiguous():
            raise ValueError("batched device data must be a contiguous (B, m, n) CUDA int32 tensor")
        bsz, m, n = data.shape
        ctx = _native.context(data.device.index)
        dev = data.device
        dp = torch.empty((bsz, m), dtype=torch.int32, device=dev)
        dq = torch.empty((bsz, n), dtype=torch.int32, device=dev)
        dr = torch.empty((bsz,), dtype=torch.int32, device=dev)
        dc = torch.empty((bsz, 4), dtype=torch.int64, device=dev) if with_counts else None
        st = ctx.lib.pluq_factor_batched(ctx.handle, data.data_ptr(), m * n, bsz, m, n, p, threshold,
                                         dp.data_ptr(), dq.data_ptr(), dr.data_ptr(),
                                         dc.data_ptr() if dc is not None else None)
        _native.raise_for(st, ctx, "pluq_batched")
        return BatchedPluq(field, data, dp, dq, dr, dc)
    arr = np.asarray(data)
    if arr.ndim != 3 or arr.dtype != np.float64 or not arr.flags.c_contiguous:
        raise ValueError("batched host data must be a contiguous (B, m, n) float64 array")
    bsz, m, n = arr.shape
    ctx = _native.context()
    psig = np.empty((bsz, m), dtype=np.int64)  # every entry is written by the call
    qsig = np.empty((bsz, n), dtype=np.int64)
    ranks = np.empty(bsz, dtype=np.int64)
    st = ctx.lib.pluq_factor_batched_host_f64(ctx.handle, arr.ctypes.data, bsz, m, n, p, threshold,
                                              _native.i64p(psig), _native.i64p(qsig), _native.i64p(ranks))
    _native.raise_for(st, ctx, "pluq_batched")
    return BatchedPluq(field, arr, psig, qsig, ranks)
