"""Single large matrix across ranks (paper_1301_4438_b200/distributed.py).

CPU: world_size-2 gloo process group; the panel kernels are a numpy stand-in backend
defined HERE (the product backend is the C ABI on each rank's GPU).  The assembled result
must equal the oracle's pluq(A) bit for bit: P = Q = I, rank, packed, and the generic
closed-form OpCounts; non-generic inputs must be detected so that rank 0 falls back to
the exact single-GPU recursion.
GPU: the CUDA backend in one process (every panel owned by rank 0) against the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import pluq_oracle as orc


class NumpyPanelBackend:
    """Test-only stand-in for CudaPanelBackend on CPU int64 torch tensors."""

    def __init__(self, p, threshold):
        self.p, self.threshold = p, threshold

    def factor_panel(self, x):
        a = x.numpy()
        f = a.astype(orc.field_dtype(self.p))
        P, Q, r, _ = orc.pluq(f, self.p, self.threshold)
        a[...] = f.astype(np.int64)
        return r, bool(np.array_equal(P, np.arange(a.shape[0]))), np.asarray(Q, dtype=np.int64)

    def trsm_llu(self, l, b):
        bb = b.numpy().astype(orc.field_dtype(self.p))
        orc.trsm_left_unit_lower(l.numpy().astype(orc.field_dtype(self.p)), bb, self.p, orc.Counts())
        b.numpy()[...] = bb.astype(np.int64)

    def gemm_sub(self, c, a, b):
        cc = c.numpy()
        cc[...] = np.mod(cc - orc.matmul_mod(a.numpy(), b.numpy(), self.p).astype(np.int64), self.p)

    def is_zero(self, x):
        return not x.numpy().any()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [  # (name, m, n, rank or None, p, width)
    ("full", 40, 40, None, 65521, 8),
    ("wide", 24, 50, None, 65521, 8),
    ("tall", 50, 24, None, 65521, 8),
    ("rank20_mid_panel", 40, 44, 20, 65521, 8),   # zero pivot inside panel 2 (owner rank 0)
    ("rank12_edge", 40, 40, 16, 65521, 8),        # zero pivot on a panel edge
    ("small_p", 36, 36, None, 101, 8),
    ("non_generic", 32, 40, 12, 101, 8),          # prescribed profiles -> not generic
]


def _matrix(name, m, n, r, p):
    if name == "non_generic":
        a, _, _ = orc.gen_cfg4(seed=2, m=m, n=n, r=r, p=p)
        return a
    if r is None:
        return np.random.default_rng(m * n + p).integers(0, p, (m, n))
    return orc.gen_xy_rank(m, n, r, p, 3)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1301_4438_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for name, m, n, r, p, width in CASES:
            a0 = _matrix(name, m, n, r, p)
            full = torch.from_numpy(a0.astype(np.int64)) if rank == 0 else None
            flags = D._Flags(torch.device("cpu"), torch.int64)
            slab = D.scatter_panels(full, m, n, width, flags.empty)
            owned = list(slab.owned)
            rk = D.distributed_generic_lu(slab, m, n, width, NumpyPanelBackend(p, 30), flags)
            if rk is not None:
                D.gather_panels(slab, full if rank == 0 else None, m, n, width, flags.empty)
            out.append((name, rk, owned, full.numpy().copy() if rank == 0 and rk is not None else None))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_distributed_panels_vs_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for i, (name, m, n, r, p, width) in enumerate(CASES):
        a0 = _matrix(name, m, n, r, p)
        x = a0.astype(orc.field_dtype(p))
        P, Q, rr, _ = orc.pluq(x, p, 30)
        generic = np.array_equal(P, np.arange(m)) and np.array_equal(Q, np.arange(n))
        npan = (n + width - 1) // width
        assert res[0][i][2] == [k for k in range(npan) if k % 2 == 0]  # block-cyclic ownership
        assert res[1][i][2] == [k for k in range(npan) if k % 2 == 1]
        rk0, rk1 = res[0][i][1], res[1][i][1]
        assert rk0 == rk1, name  # every rank reaches the same decision
        if not generic:
            assert rk0 is None, name
            continue
        assert rk0 == rr, name
        assert np.array_equal(res[0][i][3], x.astype(np.int64)), name


# ---------------------------------------------------------------------------------------
# 2D block-cyclic grid (pr x pc) over 4 gloo ranks
# ---------------------------------------------------------------------------------------

CASES_2D = [  # (name, m, n, rank or None, p, width)
    ("full", 40, 40, None, 65521, 8),
    ("wide", 24, 50, None, 65521, 8),
    ("tall", 52, 24, None, 65521, 8),
    ("ragged", 45, 43, None, 65521, 8),           # partial last row block and panel
    ("rank20_mid_panel", 40, 44, 20, 65521, 8),
    ("rank16_edge", 40, 40, 16, 65521, 8),
    ("small_p", 36, 36, None, 101, 8),
    ("non_generic", 32, 40, 12, 101, 8),
]


def _worker_2d(rank, world, port, grids, q):
    import torch
    import torch.distributed as dist

    from paper_1301_4438_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for grid in grids:
            g2 = D.Grid2D(grid[0], grid[1], rank)
            g2.make_groups()
            for name, m, n, r, p, width in CASES_2D:
                a0 = _matrix(name, m, n, r, p)
                full = torch.from_numpy(a0.astype(np.int64)) if rank == 0 else None
                flags = D._Flags(torch.device("cpu"), torch.int64)
                loc = D.scatter_2d(full, m, n, width, g2, flags.empty)
                rk = D.distributed_generic_lu_2d(loc, m, n, width, g2, NumpyPanelBackend(p, 30), flags)
                if rk is not None:
                    D.gather_2d(loc, full if rank == 0 else None, m, n, width, g2, flags.empty)
                out.append((grid, name, rk, full.numpy().copy() if rank == 0 and rk is not None else None))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_four_rank_2d_grid_vs_oracle():
    grids = [(2, 2), (4, 1), (1, 4)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_2d, args=(r, 4, port, grids, q)) for r in range(4)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    i = 0
    for grid in grids:
        for name, m, n, r, p, width in CASES_2D:
            a0 = _matrix(name, m, n, r, p)
            x = a0.astype(orc.field_dtype(p))
            P, Q, rr, _ = orc.pluq(x, p, 30)
            generic = np.array_equal(P, np.arange(m)) and np.array_equal(Q, np.arange(n))
            ranks = {res[k][i][2] for k in range(4)}
            assert len(ranks) == 1, (grid, name)  # every rank reaches the same decision
            rk0 = res[0][i][2]
            if not generic:
                assert rk0 is None, (grid, name)
            else:
                assert rk0 == rr, (grid, name)
                assert np.array_equal(res[0][i][3], x.astype(np.int64)), (grid, name)
            i += 1


# ---------------------------------------------------------------------------------------
# GPU: the CUDA backend (C ABI) in a single process, several panels on one rank
# ---------------------------------------------------------------------------------------


@pytest.mark.gpu
def test_cuda_distributed_repaired_coincidence(cuda_ok):
    """pluq_distributed on a matrix with a coincidental zero minor (the seed-0 cfg5
    structure) stays on the distributed path: the panel repair, then the replay check."""
    import torch

    import paper_1301_4438_b200 as pb
    from paper_1301_4438_b200 import distributed as D

    p, m, n, g = 65521, 600, 640, 150
    a0 = _coincidence(m, n, g, p, 5)
    x = a0.astype(np.float64)
    c0 = orc.Counts()
    P, Q, rr, _ = orc.pluq(x, p, 30, c0)
    for grid in (None, (1, 1)):
        a = pb.DenseMatrix(pb.PrimeField(p), torch.from_numpy(a0).cuda().to(torch.int32))
        c = pb.OpCounts()
        f = D.pluq_distributed(a, m, n, p, 30, width=128, counts=c, grid=grid)
        assert not D.last_info["fallback"] and D.last_info["repaired_panels"] == 1
        assert f.rank == rr and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
        assert np.array_equal(a.data.cpu().numpy().astype(np.int64), x.astype(np.int64))
        assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == c0.as_tuple()


@pytest.mark.gpu
@pytest.mark.parametrize("name,m,n,r,p,width", [
    ("full", 300, 300, None, 65521, 64), ("wide", 200, 420, None, 65521, 96),
    ("rank150", 320, 300, 150, 65521, 64), ("p23", 256, 256, None, 8388593, 64),
    ("non_generic", 200, 260, 90, 65521, 64),
])
@pytest.mark.parametrize("grid", [None, (1, 1)])
def test_cuda_panels_vs_oracle(cuda_ok, name, m, n, r, p, width, grid):
    import torch

    import paper_1301_4438_b200 as pb
    from paper_1301_4438_b200.distributed import pluq_distributed

    a0 = _matrix(name, m, n, r, p)
    x = a0.astype(orc.field_dtype(p))
    c0 = orc.Counts()
    P, Q, rr, _ = orc.pluq(x, p, 30, c0)
    a = pb.DenseMatrix(pb.PrimeField(p), torch.from_numpy(a0).cuda().to(torch.int32))
    c = pb.OpCounts()
    f = pluq_distributed(a, m, n, p, 30, width=width, counts=c, grid=grid)
    assert f.rank == rr and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(a.data.cpu().numpy().astype(np.int64), x.astype(np.int64))
    assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == \
           (c0.field_mul, c0.field_add, c0.field_inv, c0.modular_reductions)
    assert f.packed is a


# ---------------------------------------------------------------------------------------
# a coincidental zero leading minor (the seed-0 cfg5 structure): the panel holding it
# permutes only its own columns; the ranks collect that permutation and rank 0 checks the
# global rank profile matrix with the replay of Alg. 1 (pluq_rank_profile_replay)
# ---------------------------------------------------------------------------------------


def _coincidence(m, n, g, p, seed):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, p, (m, n))
    coef = rng.integers(0, p, g).astype(object)
    a[g, :g + 1] = np.array((coef @ a[:g, :g + 1].astype(object)) % p, dtype=np.int64)
    return a


COINC = [("inside_panel", 40, 44, 11), ("second_rank_panel", 40, 40, 19), ("last_row_panel", 32, 40, 29)]


def _worker_coinc(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1301_4438_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for grid in (None, (2, 1), (1, 2)):
            for name, m, n, g in COINC:
                p, width = 65521, 8
                a0 = _coincidence(m, n, g, p, g)
                full = torch.from_numpy(a0.astype(np.int64)) if rank == 0 else None
                flags = D._Flags(torch.device("cpu"), torch.int64)
                colperm = []
                if grid is None:
                    slab = D.scatter_panels(full, m, n, width, flags.empty)
                    rk = D.distributed_generic_lu(slab, m, n, width, NumpyPanelBackend(p, 30), flags, colperm)
                    if rk is not None:
                        D.gather_panels(slab, full if rank == 0 else None, m, n, width, flags.empty)
                else:
                    g2 = D.Grid2D(grid[0], grid[1], rank)
                    g2.make_groups()
                    loc = D.scatter_2d(full, m, n, width, g2, flags.empty)
                    rk = D.distributed_generic_lu_2d(loc, m, n, width, g2, NumpyPanelBackend(p, 30), flags, colperm)
                    if rk is not None:
                        D.gather_2d(loc, full if rank == 0 else None, m, n, width, g2, flags.empty)
                out.append((grid, name, rk, [(c0, qq.tolist()) for c0, qq in colperm],
                            full.numpy().copy() if rank == 0 and rk is not None else None))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_column_repairs_vs_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_coinc, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    i = 0
    for grid in (None, (2, 1), (1, 2)):
        for name, m, n, g in COINC:
            p = 65521
            a0 = _coincidence(m, n, g, p, g)
            x = a0.astype(np.float64)
            P, Q, rr, _ = orc.pluq(x, p, 30)
            assert np.array_equal(P, np.arange(m)) and not np.array_equal(Q, np.arange(n)), name
            r0, r1 = res[0][i], res[1][i]
            assert r0[2] == r1[2] == rr and r0[3] == r1[3], (grid, name)  # same decision and repairs
            sig = np.arange(n)
            for c0, qq in r0[3]:
                sig[c0:c0 + len(qq)] = c0 + np.asarray(qq)
            assert np.array_equal(sig, Q), (grid, name)
            assert np.array_equal(r0[4], x.astype(np.int64)), (grid, name)
            i += 1
