"""Every tuning option of the CUDA path gives the reference's bits (A/B of the kernel variants).

The defaults are exercised by test_gpu_parity.py; here each alternative kernel selected by
an option is run against the oracle on inputs that reach it: non-generic 64x64 batch
blocks (rank-profile kernel: lazy phases, parallel symbolic replay), cfg4-shaped leaves
(shape-2 rank-profile kernel), 128-wide speculative blocks (diagonal kernels, parallel
panel solves) and the tensor-core GEMM (MN-major vs transposed B operand).
"""

import numpy as np
import pytest

from oracle import pluq_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda_ok):
    import paper_1301_4438_b200 as mod
    from paper_1301_4438_b200 import _native

    _native.load_library()
    return mod


def _oracle(a0, p, thr=30):
    x = np.asarray(a0, dtype=np.int64).astype(orc.field_dtype(p))
    c = orc.Counts()
    P, Q, r, c = orc.pluq(x, p, thr, c)
    return P, Q, r, x.astype(np.int64), c.as_tuple()


DEFAULTS = {"sym_par": 1, "rpm_lazy": 1, "diag_lazy": 4, "tc_mnb": 1, "par_trsm": 1, "tc_trsm": 1,
            "pair_leaves": 1, "stream_fb": 4, "fb_prefix": 1, "rpm_eager": 1, "small_cap": 128 * 128}


class _opts:
    def __init__(self, **kw):
        from paper_1301_4438_b200 import _native

        self.ctx, self.kw = _native.context(), kw

    def __enter__(self):
        self.old = {k: self.ctx.get_option(k) for k in self.kw}
        for k, v in self.kw.items():
            self.ctx.set_option(k, v)

    def __exit__(self, *exc):
        for k, v in self.old.items():
            self.ctx.set_option(k, v)


def _nongeneric_batch(p, n_blocks, seed):
    """64x64 blocks whose rank profile is not generic (zero leading minors, low rank)."""
    rng = np.random.default_rng(seed)
    out = []
    for b in range(n_blocks):
        kind = b % 3
        if kind == 0:
            a = rng.integers(0, p, (64, 64))
            a[int(rng.integers(0, 64))] = 0  # a zero row
            a[:, int(rng.integers(0, 8))] = 0  # a zero leading column
        elif kind == 1:
            a = orc.gen_xy_rank(64, 64, int(rng.integers(1, 60)), p, seed + b)
        else:
            a, _, _ = orc.gen_cfg4(seed=seed + b, m=64, n=64, r=int(rng.integers(4, 40)), p=p)
        out.append(np.asarray(a, dtype=np.int64))
    return np.stack(out)


@pytest.mark.parametrize("opts", [dict(sym_par=0), dict(rpm_lazy=0), dict(sym_par=0, rpm_lazy=0), dict(fb_prefix=0),
                                  dict(rpm_eager=0), dict(rpm_eager=0, fb_prefix=0), {}])
@pytest.mark.parametrize("p", [65521, 8388593, 101])
def test_rank_profile_kernel_variants(pb, opts, p):
    import torch

    batch = _nongeneric_batch(p, 24, seed=31 + p % 97)
    with _opts(**opts):
        t = torch.from_numpy(batch).cuda().to(torch.int32)
        res = pb.pluq_batched(t, p, 30, with_counts=True)
        torch.cuda.synchronize()
    counts = res.counts.cpu().numpy()
    for b in range(batch.shape[0]):
        P, Q, r, packed, cnt = _oracle(batch[b], p)
        assert int(res.ranks[b]) == r
        assert np.array_equal(res.p_sigma[b].cpu().numpy(), P)
        assert np.array_equal(res.q_sigma[b].cpu().numpy(), Q)
        assert np.array_equal(t[b].cpu().numpy(), packed)
        assert tuple(int(v) for v in counts[b]) == cnt


@pytest.mark.parametrize("opts", [dict(sym_par=0), dict(rpm_lazy=0), dict(pair_leaves=0), dict(rpm_eager=0), {}])
@pytest.mark.parametrize("thr", [30, 4])
def test_cfg4_shaped_leaves(pb, opts, thr):
    """Prescribed rank profiles: the host recursion ends in shape-2 rank-profile leaves."""
    p = 8388593
    a0, _, _ = orc.gen_cfg4(seed=5, m=200, n=320, r=90, p=p)
    P, Q, r, packed, cnt = _oracle(a0, p, thr)
    with _opts(**opts):
        a = pb.DenseMatrix(pb.PrimeField(p), np.asarray(a0, dtype=np.int64))
        c = pb.OpCounts()
        f = pb.pluq(a, threshold=thr, counts=c)
    assert f.rank == r
    assert np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(np.asarray(a.data, dtype=np.int64), packed)
    assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == cnt


@pytest.mark.parametrize("opts", [dict(diag_lazy=1), dict(diag_lazy=3), dict(par_trsm=0), dict(diag_lazy=1, par_trsm=0), dict(tc_trsm=0), {}])
@pytest.mark.parametrize("case", [("full", 400, 400, None), ("rank200", 400, 380, 200), ("rank128", 384, 384, 128),
                                  ("rank77", 300, 330, 77), ("rank129", 260, 300, 129)])
def test_speculative_variants(pb, opts, case):
    name, m, n, r = case
    p = 65521
    rng = np.random.default_rng(m + n)
    a0 = rng.integers(0, p, (m, n)) if r is None else orc.gen_xy_rank(m, n, r, p, 11)
    P, Q, rk, packed, _ = _oracle(a0, p)
    with _opts(small_cap=1, **opts):
        a = pb.DenseMatrix(pb.PrimeField(p), np.asarray(a0, dtype=np.int64))
        f = pb.pluq(a)
        st = pb.last_stats()
    assert st["speculative_ok"] >= 1
    assert f.rank == rk
    assert np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(np.asarray(a.data, dtype=np.int64), packed)


@pytest.mark.parametrize("mnb,epi,cfg", [(0, 8, 1), (1, 8, 1), (1, 16, 1), (1, 8, 2)],
                         ids=["kmajorB", "mnB", "mnB_epi16", "mnB_twopass"])
@pytest.mark.parametrize("shape", [(256, 384, 200), (130, 260, 1100), (512, 128, 64), (1000, 700, 2048),
                                   (300, 1300, 2500)])
def test_tc_gemm_b_layouts(pb, mnb, shape, epi, cfg):
    import torch
    from paper_1301_4438_b200 import _native

    m, n, k = shape
    p = 65521
    rng = np.random.default_rng(m * 7 + k)
    A = rng.integers(0, p, (m, k))
    B = rng.integers(0, p, (k, n))
    C = rng.integers(0, p, (m, n))
    tc = torch.from_numpy(C).cuda().to(torch.int32)
    ta = torch.from_numpy(A).cuda().to(torch.int32)
    tb = torch.from_numpy(B).cuda().to(torch.int32)
    with _opts(tc_mnb=mnb, tc_epi=epi, tc_cfg=cfg):
        ctx = _native.context()
        st = ctx.lib.pluq_modgemm_sub_tc(ctx.handle, tc.data_ptr(), n, ta.data_ptr(), k, tb.data_ptr(), n, m, n, k, p)
        _native.raise_for(st, ctx, "tc gemm")
        torch.cuda.synchronize()
    want = (C - orc._mulmod_exact(A, B, p)) % p
    assert np.array_equal(tc.cpu().numpy().astype(np.int64), want.astype(np.int64))


@pytest.mark.parametrize("p", [65521, 101, 8388593])
@pytest.mark.parametrize("shape", [(128, 128), (96, 80), (40, 128), (128, 24)])
def test_batched_nongeneric_shapes(pb, p, shape):
    """Non-generic batches beyond 64x64: rank-profile kernel shape 2 (lazy phases with and
    without the shared-memory inverse table) and the runtime-shape generic kernel."""
    import torch

    m, n = shape
    rng = np.random.default_rng(m * 1000 + n + p % 997)
    blocks = []
    for b in range(6):
        if b % 3 == 0:
            a = rng.integers(0, p, (m, n))
            a[:, :3] = 0  # zero leading columns: not generic
        elif b % 3 == 1:
            a = orc.gen_xy_rank(m, n, int(rng.integers(1, min(m, n))), p, b + 5)
        else:
            a = rng.integers(0, p, (m, n))  # generic w.h.p.
        blocks.append(np.asarray(a, dtype=np.int64))
    batch = np.stack(blocks)
    t = torch.from_numpy(batch).cuda().to(torch.int32)
    res = pb.pluq_batched(t, p, 30, with_counts=True)
    torch.cuda.synchronize()
    counts = res.counts.cpu().numpy()
    for b in range(batch.shape[0]):
        P, Q, r, packed, cnt = _oracle(batch[b], p)
        assert int(res.ranks[b]) == r, b
        assert np.array_equal(res.p_sigma[b].cpu().numpy(), P), b
        assert np.array_equal(res.q_sigma[b].cpu().numpy(), Q), b
        assert np.array_equal(t[b].cpu().numpy(), packed), b
        assert tuple(int(v) for v in counts[b]) == cnt, b


@pytest.mark.parametrize("prefix", [1, 0])
@pytest.mark.parametrize("stream_fb", [0, 4, 1])
def test_streaming_fallback_consumer(pb, stream_fb, prefix):
    """Large batches: the rank-profile consumer runs concurrently with the generic kernel
    (stream_fb CTAs claiming the failure list) or after it (0) — same bits either way."""
    import torch

    p = 65521
    rng = np.random.default_rng(2024 + stream_fb)
    batch = rng.integers(0, p, (2048, 64, 64))
    bad = rng.choice(2048, 40, replace=False)
    for k, b in enumerate(bad):
        if k % 4 == 3:
            batch[b] = orc.gen_xy_rank(64, 64, 63, p, int(b))  # generic up to the last pivot
        elif k % 2:
            batch[b] = orc.gen_xy_rank(64, 64, int(rng.integers(1, 63)), p, int(b))
        else:
            batch[b][:, 0] = 0  # zero leading column: not generic
    with _opts(stream_fb=stream_fb, fb_prefix=prefix):
        t = torch.from_numpy(batch).cuda().to(torch.int32)
        res = pb.pluq_batched(t, p, 30, with_counts=True)
        torch.cuda.synchronize()
    counts = res.counts.cpu().numpy()
    check = sorted(set(bad.tolist()) | set(rng.choice(2048, 24, replace=False).tolist()))
    for b in check:
        P, Q, r, packed, cnt = _oracle(batch[b], p)
        assert int(res.ranks[b]) == r, b
        assert np.array_equal(res.p_sigma[b].cpu().numpy(), P), b
        assert np.array_equal(res.q_sigma[b].cpu().numpy(), Q), b
        assert np.array_equal(t[b].cpu().numpy(), packed), b
        assert tuple(int(v) for v in counts[b]) == cnt, b


def test_prefix_slots_overflow(pb):
    """More failing blocks than prefix slots (1024): the blocks beyond the pool are
    factored from scratch by the rank-profile kernel; every block still matches."""
    import torch

    p = 65521
    rng = np.random.default_rng(99)
    nb = 1300
    batch = rng.integers(0, p, (nb, 64, 64))
    for b in range(nb):  # every block fails somewhere: zero column c (pivot c is zero)
        batch[b][:, int(rng.integers(0, 64))] = 0
    t = torch.from_numpy(batch).cuda().to(torch.int32)
    res = pb.pluq_batched(t, p, 30)
    torch.cuda.synchronize()
    for b in list(range(0, nb, 37)) + list(range(nb - 12, nb)):
        P, Q, r, packed, _ = _oracle(batch[b], p)
        assert int(res.ranks[b]) == r, b
        assert np.array_equal(res.p_sigma[b].cpu().numpy(), P), b
        assert np.array_equal(res.q_sigma[b].cpu().numpy(), Q), b
        assert np.array_equal(t[b].cpu().numpy(), packed), b
