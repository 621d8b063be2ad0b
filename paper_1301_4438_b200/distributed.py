"""One large matrix across ranks: block-column distributed generic-profile LU.

SURVEY §8(e) / BASELINE north star: for a single large matrix the trailing
Schur-complement update is partitioned across GPUs and the pivot panels are broadcast
(NCCL over NVLink on the GPU box, gloo in the CPU tests); the recursion and the base case
stay on one GPU.

Layout (default): column panels of width W, panel k (columns [kW, kW+W)) owned by rank
k % N for all m rows (a 1 x N process grid); grid=(pr, pc) selects the 2D block-cyclic
layout below (`distributed_generic_lu_2d`).  Step k of the 1 x N layout:
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

# outcome of the last pluq_distributed on this rank 0: {"fallback": bool, "repaired_panels": int}
last_info: dict = {}


class CudaPanelBackend:
    """Panel operations on CUDA int32 tensors through the C ABI (this rank's device)."""

    def __init__(self, p: int, threshold: int, device: int):
        self.p, self.threshold, self.device = int(p), int(threshold), device
        self.ctx = _native.context(device)
        self.lib = self.ctx.lib

    def factor_panel(self, x):
        """In-place exact PLUQ of a contiguous panel; returns (rank, rows_in_order, Q.sigma):
        rows_in_order means P = I, and then the panel holds the LU of panel[:, Q]."""
        m, n = x.shape
        P = np.empty(m, np.int64)
        Q = np.empty(n, np.int64)
        r = np.zeros(1, np.int64)
        c = np.zeros(4, np.int64)
        st = self.lib.pluq_factor(self.ctx.handle, x.data_ptr(), x.stride(0), m, n, self.p, self.threshold,
                                  _native.i64p(P), _native.i64p(Q), _native.i64p(r), _native.i64p(c))
        _native.raise_for(st, self.ctx, "pluq_factor (panel)")
        return int(r[0]), bool(np.array_equal(P, np.arange(m))), Q

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


def _panel_verdict(res, wk: int, colperm):
    """(rank, usable, q) from a backend's factor_panel result.  A panel is usable when its
    rows stay in order (P = I) and, unless column repairs are collected (colperm is a list),
    its columns too.  q: the panel's Q.sigma when it is not the identity, else None."""
    if len(res) == 2:  # legacy backends: (rank, generic)
        return int(res[0]), bool(res[1]), None
    rk, rows_ok, q = res
    q = None if q is None or np.array_equal(np.asarray(q), np.arange(wk)) else np.asarray(q, dtype=np.int64)
    usable = bool(rows_ok) and (q is None or colperm is not None)
    return int(rk), usable, q


def _share_q(q, wk: int, owner: int, flags, colperm, c0: int, world: int) -> None:
    """Broadcast a repaired panel's column permutation and record it (global indices)."""
    import torch
    import torch.distributed as dist

    buf = torch.zeros(wk, dtype=torch.int64, device=flags.device)
    if q is not None:
        buf.copy_(torch.from_numpy(q))
    if world > 1:
        dist.broadcast(buf, src=owner)
    colperm.append((c0, buf.cpu().numpy().astype(np.int64)))
    return buf


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


def distributed_generic_lu(slab: LocalSlab, m: int, n: int, width: int, backend, flags, colperm=None,
                           lookahead: bool = True, prefetch: bool = True):
    """Factor the distributed panels in place.  Returns the rank r when the matrix has a
    generic rank profile (then P = Q = I), or None when it does not (panels are then
    partially updated; the caller restarts from the original on one GPU).

    colperm (a list) also accepts panels whose factorization permuted only their own
    columns (the pivot repair of a coincidental zero minor, csrc speculative_lu): the panel
    then holds the LU of its columns in that order, later steps only use its L part, and
    (c0, Q.sigma) is appended for the caller's check of the global rank profile matrix.

    lookahead: the owner of panel k+1 updates that panel's columns with panel k FIRST, factors
    it, and only then updates the rest of its later panels, so the factorization of k+1 hides
    behind the other ranks' trailing updates (the HPL look-ahead); collectives keep the same
    order on every rank.

    prefetch (with lookahead): the broadcast of panel k+1 is started asynchronously during step
    k — by its owner right after the look-ahead factorization, by the other ranks before their
    own trailing update — and waited for at the start of step k+1, so the panel transfer
    overlaps the tensor-core update instead of preceding it (NCCL runs it on its own stream)."""
    import torch.distributed as dist

    rank, world = _world()
    mn = min(m, n)
    bounds = [b for b in panel_bounds(n, width) if b[0] < mn]

    def factor(k):
        c0, c1 = bounds[k]
        return _panel_verdict(backend.factor_panel(slab.panel(k)[c0:, :]), c1 - c0, colperm)

    def post(k1, res):
        """Start the broadcast of panel k1 (verdict flag + factored panel) without waiting for
        it: the owner passes its verdict, the other ranks post the matching receives.  The
        collectives are issued in the same order on every rank."""
        c0n, c1n = bounds[k1]
        own = panel_owner(k1, world)
        flag = flags()
        pan = flags.new_panel(m - c0n, c1n - c0n)  # contiguous broadcast buffer
        q = None
        if rank == own:
            rk, generic, q = res
            pan.copy_(slab.panel(k1)[c0n:, :])
            flag[0], flag[1] = rk, int(generic) + 2 * int(q is not None)
        works = []
        if world > 1:
            works.append(dist.broadcast(flag, src=own, async_op=True))
            works.append(dist.broadcast(pan, src=own, async_op=True))
        return flag, pan, q, works

    ahead = factor(0) if bounds and rank == panel_owner(0, world) else None
    pending = None  # panel k's broadcast, started during step k - 1 (prefetch)
    for k, (c0, c1) in enumerate(bounds):
        owner = panel_owner(k, world)
        wk = c1 - c0
        if pending is None:
            res = (ahead if ahead is not None else factor(k)) if rank == owner else None
            ahead = None
            pending = post(k, res)
        flag, pan, q, works = pending
        pending = None
        for w in works:
            w.wait()
        rk, generic, repaired = int(flag[0]), bool(int(flag[1]) & 1), bool(int(flag[1]) & 2)
        if not generic:
            return None
        if repaired:
            qt = _share_q(q, wk, owner, flags, colperm, c0, world)
            if rank == owner and c0 > 0:  # the U rows of earlier pivots in these columns move too
                top = slab.panel(k)[:c0, :]
                top.copy_(top[:, qt.to(top.device)])
        g = c0 + rk
        rest = slab.after(k)
        # look-ahead + prefetch: the owner of panel k+1 brings that panel up to date first,
        # factors it and starts its broadcast; the other ranks post the receive BEFORE their own
        # trailing update, so the transfer of panel k+1 runs under the update with panel k
        la_step = lookahead and rk == wk and k + 1 < len(bounds)
        nxt = panel_owner(k + 1, world) if la_step else -1
        if la_step and prefetch and rank != nxt:
            pending = post(k + 1, None)
        if rest is not None and rk > 0:
            la = la_step and rank == nxt
            w1 = slab.w[k + 1] if la else 0
            parts = [(0, w1), (w1, rest.shape[1])] if la else [(0, rest.shape[1])]
            for i, (a0, a1) in enumerate(parts):
                if a1 > a0:
                    top = rest[c0:g, a0:a1]
                    backend.trsm_llu(pan[:rk, :rk], top)                          # U12 rows
                    if g < m:
                        backend.gemm_sub(rest[g:, a0:a1], pan[rk:, :rk], top)  # A22 -= L21 U12
                if la and i == 0:
                    ahead = factor(k + 1)  # panel k+1 is up to date: factor it now
                    if prefetch:
                        pending = post(k + 1, ahead)
                        ahead = None
        if rk < wk:
            # zero pivot at g: generic only if the whole Schur complement A[g:, g:] vanishes
            # (panel k's own part was checked by the exact panel factorization)
            nz = flags()
            nz[0] = int(rest is not None and g < m and not backend.is_zero(rest[g:, :]))
            if world > 1:
                dist.all_reduce(nz, op=dist.ReduceOp.MAX)
            return g if int(nz[0]) == 0 else None
    return mn


# ---------------------------------------------------------------------------------------
# 2D block-cyclic process grid (pr x pc): W x W blocks, row block b on grid row b % pr,
# column panel k on grid column k % pc.  Per panel step the panel column is gathered on
# its diagonal owner and factored there (the recursion and base case stay on one GPU),
# the factored panel is broadcast, the grid row holding the pivot rows solves U12 for its
# columns and broadcasts it down each grid column, and every rank updates its own rows x
# columns with one GEMM (A22 -= L21 U12): the Schur-complement update is 2D-partitioned.
# ---------------------------------------------------------------------------------------


class Grid2D:
    def __init__(self, pr: int, pc: int, rank: int):
        self.pr, self.pc = pr, pc
        self.gr, self.gc = divmod(rank, pc)
        self.col_groups = None

    def rank_of(self, gr: int, gc: int) -> int:
        return gr * self.pc + gc

    def make_groups(self):
        """One process group per grid column (every rank creates every group, in order)."""
        import torch.distributed as dist

        self.col_groups = [dist.new_group([self.rank_of(r, c) for r in range(self.pr)]) for c in range(self.pc)]


def _row_blocks(m: int, width: int, gr: int, pr: int):
    """(global start, global end, local start) of the row blocks grid row gr owns."""
    out, loc = [], 0
    for b, r0 in enumerate(range(0, m, width)):
        if b % pr == gr:
            r1 = min(r0 + width, m)
            out.append((r0, r1, loc))
            loc += r1 - r0
    return out, loc


class LocalBlocks:
    """A rank's blocks of the 2D layout in one dense tensor: its row blocks (in order) x
    its column panels (in order), so that "my rows >= g" and "my panels > k" are always a
    contiguous row suffix and column suffix."""

    def __init__(self, tensor, rows, cols: LocalSlab):
        self.t, self.rows, self.cols = tensor, rows, cols

    def first_row_at_or_after(self, g: int) -> int:
        for r0, r1, l0 in self.rows:
            if r1 > g:
                return l0 + max(0, g - r0)
        return self.t.shape[0]

    def global_rows(self, from_local: int):
        """Global indices of the local rows [from_local, end) as an int64 numpy array."""
        parts = [np.arange(max(r0, r0 + from_local - l0), r1, dtype=np.int64)
                 for r0, r1, l0 in self.rows if l0 + (r1 - r0) > from_local]
        return np.concatenate(parts) if parts else np.zeros(0, np.int64)

    def panel(self, k):
        return self.t[:, self.cols.off[k]:self.cols.off[k] + self.cols.w[k]]

    def after(self, k):
        later = [j for j in self.cols.owned if j > k]
        return None if not later else self.t[:, self.cols.off[later[0]]:]


def _layout_2d(m, n, width, grid: Grid2D, gr=None, gc=None):
    gr = grid.gr if gr is None else gr
    gc = grid.gc if gc is None else gc
    rows, nrows = _row_blocks(m, width, gr, grid.pr)
    owned, offsets, widths, ncols = _layout(n, width, gc, grid.pc)
    return rows, nrows, LocalSlab(None, owned, offsets, widths), ncols


def _index_lists(m, n, width, grid, gr, gc):
    rows, _, cols, _ = _layout_2d(m, n, width, grid, gr, gc)
    ridx = [i for r0, r1, _ in rows for i in range(r0, r1)]
    cidx = [j for k in cols.owned for j in range(panel_bounds(n, width)[k][0], panel_bounds(n, width)[k][1])]
    return ridx, cidx


def scatter_2d(a_full, m, n, width, grid: Grid2D, make_empty) -> LocalBlocks:
    import torch
    import torch.distributed as dist

    rank, world = _world()
    rows, nrows, cols, ncols = _layout_2d(m, n, width, grid)
    loc = LocalBlocks(make_empty(nrows, ncols), rows, cols)
    for dst in range(world):
        gr, gc = divmod(dst, grid.pc)
        ridx, cidx = _index_lists(m, n, width, grid, gr, gc)
        if not ridx or not cidx:
            continue
        if rank == 0:
            ri = torch.tensor(ridx, device=a_full.device)
            ci = torch.tensor(cidx, device=a_full.device)
            blk = a_full.index_select(0, ri).index_select(1, ci).contiguous()
            if dst == 0:
                loc.t.copy_(blk)
            else:
                dist.send(blk, dst=dst)
        elif rank == dst:
            dist.recv(loc.t, src=0)
    return loc


def gather_2d(loc: LocalBlocks, a_full, m, n, width, grid: Grid2D, make_empty):
    import torch
    import torch.distributed as dist

    rank, world = _world()
    for src in range(world):
        gr, gc = divmod(src, grid.pc)
        ridx, cidx = _index_lists(m, n, width, grid, gr, gc)
        if not ridx or not cidx:
            continue
        if rank == 0:
            if src == 0:
                blk = loc.t
            else:
                blk = make_empty(len(ridx), len(cidx))
                dist.recv(blk, src=src)
            ri = torch.tensor(ridx, device=a_full.device)
            ci = torch.tensor(cidx, device=a_full.device)
            a_full[ri.unsqueeze(1), ci.unsqueeze(0)] = blk
        elif rank == src:
            dist.send(loc.t.contiguous(), dst=0)


def distributed_generic_lu_2d(loc: LocalBlocks, m: int, n: int, width: int, grid: Grid2D, backend, flags,
                              colperm=None):
    """distributed_generic_lu on a pr x pc grid (same contract: the rank r, or None; the
    same column-repair collection through colperm)."""
    import torch
    import torch.distributed as dist

    rank, world = _world()
    mn = min(m, n)
    for k, (c0, c1) in enumerate(panel_bounds(n, width)):
        if c0 >= mn:
            break
        wk = c1 - c0
        gck, grk = k % grid.pc, k % grid.pr
        root = grid.rank_of(grk, gck)
        # 1. gather panel column k (rows >= c0) on its diagonal owner, in global row order
        pan = flags.new_panel(m - c0, wk)
        if grid.gc == gck:
            lr = loc.first_row_at_or_after(c0)
            mine = loc.panel(k)[lr:, :]
            grows = loc.global_rows(lr)
        for gr in range(grid.pr):
            src = grid.rank_of(gr, gck)
            rows_gr, _ = _row_blocks(m, width, gr, grid.pr)
            parts = [np.arange(max(r0, c0), r1, dtype=np.int64) for r0, r1, _ in rows_gr if r1 > c0]
            gidx = np.concatenate(parts) if parts else np.zeros(0, np.int64)
            if not len(gidx):
                continue
            if rank == root:
                if src == root:
                    blk = mine
                else:
                    blk = flags.new_panel(len(gidx), wk)
                    dist.recv(blk, src=src)
                if len(gidx) == gidx[-1] - gidx[0] + 1:  # contiguous rows: a slice copy
                    pan[int(gidx[0]) - c0:int(gidx[-1]) + 1 - c0] = blk
                else:
                    pan[torch.from_numpy(gidx - c0).to(pan.device)] = blk
            elif rank == src:
                dist.send(mine.contiguous(), dst=root)
        # 2. factor on the root, broadcast the verdict and the factored panel
        flag = flags()
        q = None
        if rank == root:
            rk, generic, q = _panel_verdict(backend.factor_panel(pan), wk, colperm)
            flag[0], flag[1] = rk, int(generic) + 2 * int(q is not None)
        if world > 1:
            dist.broadcast(flag, src=root)
        rk, generic, repaired = int(flag[0]), bool(int(flag[1]) & 1), bool(int(flag[1]) & 2)
        if not generic:
            return None
        if repaired:
            qt = _share_q(q, wk, root, flags, colperm, c0, world)
            if grid.gc == gck:  # the U rows of earlier pivots in these columns move too
                lr0 = loc.first_row_at_or_after(c0)
                if lr0 > 0:
                    top = loc.panel(k)[:lr0, :]
                    top.copy_(top[:, qt.to(top.device)])
        if world > 1:
            dist.broadcast(pan, src=root)
        g = c0 + rk
        # 3. the panel's grid column takes its rows of the factored panel back
        if grid.gc == gck and len(grows):
            if len(grows) == grows[-1] - grows[0] + 1:
                loc.panel(k)[lr:, :] = pan[int(grows[0]) - c0:int(grows[-1]) + 1 - c0]
            else:
                loc.panel(k)[lr:, :] = pan[torch.from_numpy(grows - c0).to(pan.device)]
        # 4. U12 on the grid row of the pivot rows, broadcast down each grid column
        rest = loc.after(k)
        top = None
        if rest is not None and rk > 0:
            if grid.gr == grk:
                t0 = loc.first_row_at_or_after(c0)
                top = rest[t0:t0 + rk, :]
                backend.trsm_llu(pan[:rk, :rk], top)
            if grid.pr > 1:
                buf = top.contiguous() if grid.gr == grk else flags.new_panel(rk, rest.shape[1])
                dist.broadcast(buf, src=grid.rank_of(grk, grid.gc), group=grid.col_groups[grid.gc])
                top = buf
            # 5. A22 -= L21 U12 on my rows >= g x my later panels
            lg = loc.first_row_at_or_after(g)
            if lg < loc.t.shape[0]:
                gl = loc.global_rows(lg)
                if len(gl) == gl[-1] - gl[0] + 1:
                    l21 = pan[int(gl[0]) - c0:int(gl[-1]) + 1 - c0, :rk]
                else:
                    l21 = pan[torch.from_numpy(gl - c0).to(pan.device)][:, :rk].contiguous()
                backend.gemm_sub(rest[lg:, :], l21, top)
        if rk < wk:
            nz = flags()
            lg = loc.first_row_at_or_after(g)
            nz[0] = int(rest is not None and lg < loc.t.shape[0] and not backend.is_zero(rest[lg:, :]))
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
                     device=None, grid: tuple[int, int] | None = None):
    """pluq() of one large matrix held by rank 0 (CUDA int32 DenseMatrix), with the
    trailing updates spread over every rank of the default process group.  All ranks call
    it; rank 0 gets the PluqFactors (in place, `f.packed is a`), the others get the rank.
    grid=(pr, pc) with pr * pc == world selects the 2D block-cyclic layout (W x W blocks);
    the default is the 1 x N column-panel layout."""
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
    colperm: list = []  # (c0, Q.sigma) of panels whose factorization repaired a zero minor
    if rank == 0:
        x = a.data
        if tuple(x.shape) != (m, n):
            raise ValueError("shape mismatch")
        full = x.clone()  # the original stays untouched until the final gather
    else:
        full = None
    if grid is not None:
        pr, pc = grid
        if pr * pc != world:
            raise ValueError("grid must cover the process group")
        g2 = Grid2D(pr, pc, rank)
        if world > 1:
            g2.make_groups()
        loc = scatter_2d(full, m, n, width, g2, flags.empty)
        r = distributed_generic_lu_2d(loc, m, n, width, g2, backend, flags, colperm)
        if r is not None:
            gather_2d(loc, full if rank == 0 else None, m, n, width, g2, flags.empty)
    else:
        slab = scatter_panels(full, m, n, width, flags.empty)
        r = distributed_generic_lu(slab, m, n, width, backend, flags, colperm)
        if r is not None:
            gather_panels(slab, full if rank == 0 else None, m, n, width, flags.empty)
    if rank != 0:
        return r
    q_sig = np.arange(n, dtype=np.int64)
    c = np.zeros(4, np.int64)
    lib = _native.load_library()
    if r is not None and colperm:
        # the panels' column repairs compose into sigma; R_A = {(k, sigma(k))} (rows in
        # order), and the result is the reference's exactly when Alg.1 replayed on R_A gives
        # P = I and Q = sigma (csrc speculative_lu, fact (2)) -- else the exact fallback
        for c0, q in colperm:
            q_sig[c0:c0 + len(q)] = c0 + q
        P = np.zeros(m, np.int64)
        Q = np.zeros(n, np.int64)
        prow = np.arange(r, dtype=np.int64)
        pcol = np.ascontiguousarray(q_sig[:r])
        st = lib.pluq_rank_profile_replay(m, n, threshold, r, _native.i64p(prow), _native.i64p(pcol),
                                          _native.i64p(P), _native.i64p(Q), _native.i64p(c))
        if st != 0 or not (np.array_equal(P, np.arange(m)) and np.array_equal(Q, q_sig)):
            r = None
    last_info.update(fallback=r is None, repaired_panels=len(colperm))
    if r is None:  # not generic: the exact recursion on one GPU, from the untouched original
        from .recursive import pluq

        return pluq(a, threshold=threshold, counts=counts)
    a.data.copy_(full)
    if counts is not None:
        if not colperm:
            _native.raise_for(lib.pluq_generic_counts(m, n, r, threshold, _native.i64p(c)), None,
                              "pluq_generic_counts")
        counts.field_mul += int(c[0]); counts.field_add += int(c[1])
        counts.field_inv += int(c[2]); counts.modular_reductions += int(c[3])
    return PluqFactors(Permutation(np.arange(m, dtype=np.int64)), Permutation(q_sig), r, a)
