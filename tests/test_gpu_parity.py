"""Parity of the CUDA path (via the C ABI) against the reference goldens and the oracle."""

import hashlib

import numpy as np
import pytest

from oracle import pluq_oracle as orc

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def pb(cuda_ok):
    import paper_1301_4438_b200 as mod
    from paper_1301_4438_b200 import _native

    _native.load_library()
    return mod


def _check(f, a_after, P, Q, r, packed, counts=None, c=None):
    assert f.rank == r
    assert np.array_equal(f.p_perm.sigma, P)
    assert np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(np.asarray(a_after, dtype=np.int64), np.asarray(packed, dtype=np.int64))
    if counts is not None:
        assert [c.field_mul, c.field_add, c.field_inv, c.modular_reductions] == list(counts)


# ---------------------------------------------------------------------------------------
# golden fixtures produced by the reference itself
# ---------------------------------------------------------------------------------------


def test_every_golden_host_buffers(pb, golden):
    """pluq()/pluq_iterative() on host DenseMatrix (e2e path) == reference, incl. OpCounts."""
    z, man = golden
    bad = []
    for e in man:
        k, p = e["key"], e["p"]
        field = pb.PrimeField(p)
        a = pb.DenseMatrix(field, z[k + "_in"])
        c = pb.OpCounts()
        f = pb.pluq_iterative(a, c) if e["route"] == "iterative" else pb.pluq(a, threshold=e["threshold"], counts=c)
        ok = (f.rank == e["rank"] and np.array_equal(f.p_perm.sigma, z[k + "_P"])
              and np.array_equal(f.q_perm.sigma, z[k + "_Q"]) and _sha(a.data) == e["packed_sha256"]
              and [c.field_mul, c.field_add, c.field_inv, c.modular_reductions] == e["counts"]
              and f.packed is a and a.data.dtype == field.dtype)
        if not ok:
            bad.append((k, e["tag"], e["route"], e["m"], e["n"], p))
    assert not bad, bad[:10]


def test_golden_device_resident(pb, golden):
    """Zero-copy path: CUDA int32 tensors in, packed result left on the device."""
    import torch

    z, man = golden
    for e in man[::5]:
        if e["route"] != "recursive":
            continue
        k, p = e["key"], e["p"]
        t = torch.from_numpy(z[k + "_in"]).cuda().to(torch.int32)
        a = pb.DenseMatrix(pb.PrimeField(p), t)
        f = pb.pluq(a, threshold=e["threshold"])
        assert f.rank == e["rank"] and np.array_equal(f.p_perm.sigma, z[k + "_P"])
        assert _sha(t.cpu().numpy()) == e["packed_sha256"]


# ---------------------------------------------------------------------------------------
# modular GEMM: tensor-core (tcgen05 kind::i8 limbs) and CUDA-core paths
# ---------------------------------------------------------------------------------------

GEMM_CASES = [
    (65521, 256, 256, 384), (65521, 300, 200, 130), (65521, 129, 131, 33), (251, 256, 512, 256),
    (8388593, 256, 192, 300), (2147483647, 128, 128, 128), (2, 130, 140, 150), (65521, 1024, 768, 2048),
]


@pytest.mark.parametrize("p,m,n,k", GEMM_CASES)
def test_tc_gemm_vs_oracle(pb, p, m, n, k):
    import torch
    from paper_1301_4438_b200 import _native

    rng = np.random.default_rng(m * 7 + n + k)
    A, B, C = rng.integers(0, p, (m, k)), rng.integers(0, p, (k, n)), rng.integers(0, p, (m, n))
    tc, ta, tb = (torch.from_numpy(x).cuda().to(torch.int32) for x in (C, A, B))
    ctx = _native.context()
    st = ctx.lib.pluq_modgemm_sub_tc(ctx.handle, tc.data_ptr(), n, ta.data_ptr(), k, tb.data_ptr(), n, m, n, k, p)
    _native.raise_for(st, ctx, "tc")
    want = (C - orc._mulmod_exact(A, B, p)) % p
    assert np.array_equal(tc.cpu().numpy().astype(np.int64), want)


def test_tc_gemm_multi_pass_k(pb):
    """K longer than one exact pass (forced small pass) must still be exact."""
    import torch
    from paper_1301_4438_b200 import _native

    p, m, n, k = 65521, 256, 256, 1000
    rng = np.random.default_rng(9)
    A, B, C = rng.integers(0, p, (m, k)), rng.integers(0, p, (k, n)), rng.integers(0, p, (m, n))
    tc, ta, tb = (torch.from_numpy(x).cuda().to(torch.int32) for x in (C, A, B))
    ctx = _native.context()
    ctx.set_option("tc_k_pass", 256)
    try:
        st = ctx.lib.pluq_modgemm_sub_tc(ctx.handle, tc.data_ptr(), n, ta.data_ptr(), k, tb.data_ptr(), n, m, n, k, p)
        _native.raise_for(st, ctx, "tc")
    finally:
        ctx.set_option("tc_k_pass", 0)
    want = (C - orc._mulmod_exact(A, B, p)) % p
    assert np.array_equal(tc.cpu().numpy().astype(np.int64), want)


def test_tc_gemm_on_strided_views(pb):
    """Operands are sub-blocks of one matrix (the recursion's case)."""
    import torch
    from paper_1301_4438_b200 import _native

    p = 65521
    rng = np.random.default_rng(3)
    X = rng.integers(0, p, (700, 900))
    t = torch.from_numpy(X).cuda().to(torch.int32)
    c, a, b = t[300:600, 400:850], t[300:600, 5:203], t[1:199, 400:850]
    ctx = _native.context()
    st = ctx.lib.pluq_modgemm_sub_tc(ctx.handle, c.data_ptr(), 900, a.data_ptr(), 900, b.data_ptr(), 900,
                                     300, 450, 198, p)
    _native.raise_for(st, ctx, "tc")
    want = X.copy()
    want[300:600, 400:850] = (X[300:600, 400:850] - orc._mulmod_exact(X[300:600, 5:203], X[1:199, 400:850], p)) % p
    assert np.array_equal(t.cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("p,m,n,k", [(65521, 100, 70, 33), (8388593, 65, 129, 200), (2147483647, 40, 50, 60)])
def test_simt_gemm_vs_oracle(pb, p, m, n, k):
    rng = np.random.default_rng(k)
    A, B, C = rng.integers(0, p, (m, k)), rng.integers(0, p, (k, n)), rng.integers(0, p, (m, n))
    kern = pb.CudaKernels(pb.PrimeField(p, allow_large_modulus=True))
    c = C.copy()
    kern.mm_acc(c, A, B, pb.OpCounts())
    assert np.array_equal(c, (C - orc._mulmod_exact(A, B, p)) % p)


# ---------------------------------------------------------------------------------------
# kernel strategy (reference test_kernels.py restated on the CUDA kernels)
# ---------------------------------------------------------------------------------------


def test_mm_acc_against_triple_loop(pb):  # test_kernels.py:40-52
    rng = np.random.default_rng(77)
    for trial in range(150):
        p = int(rng.choice([2, 3]))
        field = pb.PrimeField(p)
        kern = pb.CudaKernels(field)
        m, k, n = (int(x) for x in rng.integers(0, 6, 3))
        a = rng.integers(0, p, (m, k)).astype(field.dtype)
        b = rng.integers(0, p, (k, n)).astype(field.dtype)
        c = rng.integers(0, p, (m, n)).astype(field.dtype)
        want = c.astype(np.int64).copy()
        for i in range(m):
            for j in range(n):
                for t in range(k):
                    want[i, j] = (want[i, j] - int(a[i, t]) * int(b[t, j])) % p
        kern.mm_acc(c, a, b, pb.OpCounts())
        assert np.array_equal(c.astype(np.int64), want), (trial, p, m, k, n)


def test_mm_acc_empty_inner_and_shapes(pb):  # test_kernels.py:29-37
    field = pb.PrimeField(7)
    kern = pb.CudaKernels(field)
    c = np.array([[1, 2], [3, 4]], dtype=np.float64)
    counts = pb.OpCounts()
    kern.mm_acc(c, np.zeros((2, 0)), np.zeros((0, 2)), counts)
    assert c.tolist() == [[1, 2], [3, 4]] and counts.modular_reductions == 0
    with pytest.raises(ValueError):
        kern.mm_acc(c, np.zeros((2, 3)), np.zeros((2, 2)), counts)


def test_mm_acc_large_modulus_int64_path(pb):  # test_kernels.py:55-68
    p = 67108859
    field = pb.PrimeField(p)
    kern = pb.CudaKernels(field)
    rng = np.random.default_rng(4)
    a = rng.integers(0, p, (4, 3000)).astype(field.dtype)
    b = rng.integers(0, p, (3000, 2)).astype(field.dtype)
    c = np.zeros((4, 2), field.dtype)
    kern.mm_acc(c, a, b, pb.OpCounts())
    for i in (0, 3):
        for j in (0, 1):
            assert int(c[i, j]) == (-sum(int(a[i, t]) * int(b[t, j]) for t in range(3000))) % p


@pytest.mark.parametrize("p", [5, 1009, 65521, 8388593])
def test_trsm_remultiplication(pb, p):  # test_kernels.py:114-134
    rng = np.random.default_rng(p)
    field = pb.PrimeField(p)
    kern = pb.CudaKernels(field)
    # the last three take the large-triangle path (full inverse + one in-place GEMM) when
    # the solved side is >= 256 wide: r = 256 exactly, r not a multiple of 64, r = 2048
    for r, n in [(1, 5), (7, 0), (33, 40), (64, 17), (65, 3), (200, 150), (256, 1100), (700, 3000), (2048, 8200)]:
        l = np.tril(rng.integers(0, p, (r, r)), -1).astype(field.dtype)
        b = rng.integers(0, p, (r, n)).astype(field.dtype)
        orig = b.astype(np.int64).copy()
        kern.trsm_left_unit_lower(l, b, pb.OpCounts())
        lfull = l.astype(np.int64) + np.eye(r, dtype=np.int64)
        assert np.array_equal(orc._mulmod_exact(lfull, b.astype(np.int64), p), orig)
        u = np.triu(rng.integers(0, p, (r, r)), 1)
        u[np.arange(r), np.arange(r)] = rng.integers(1, p, r)
        u = u.astype(field.dtype)
        b2 = rng.integers(0, p, (n, r)).astype(field.dtype)
        orig2 = b2.astype(np.int64).copy()
        kern.trsm_right_upper(b2, u, pb.OpCounts())
        assert np.array_equal(orc._mulmod_exact(b2.astype(np.int64), u.astype(np.int64), p), orig2)


def test_trsm_zero_diagonal_raises(pb):  # test_kernels.py:104-111
    field = pb.PrimeField(5)
    kern = pb.CudaKernels(field)
    counts = pb.OpCounts()
    with pytest.raises(ZeroDivisionError):
        kern.trsm_right_upper(np.zeros((2, 2)), np.array([[1.0, 2.0], [0.0, 0.0]]), counts)
    assert counts.field_inv == 0


class _Recording:
    """Wraps CudaKernels and asserts the closed-form charges of every call (test_kernels.py:137-180)."""

    def __init__(self, pb, field):
        self.k = pb.CudaKernels(field)
        self.calls = 0

    def mm_acc(self, c, a, b, counts):
        before = counts.copy()
        self.k.mm_acc(c, a, b, counts)
        m, k = a.shape
        n = b.shape[1]
        expect = m * n if (k and m and n) else 0
        assert counts.modular_reductions - before.modular_reductions == expect
        self.calls += 1

    def trsm_left_unit_lower(self, l, b, counts):
        before = counts.copy()
        self.k.trsm_left_unit_lower(l, b, counts)
        r, n = l.shape[0], b.shape[1]
        assert counts.modular_reductions - before.modular_reductions == (r * n if r and n else 0)
        self.calls += 1

    def trsm_right_upper(self, b, u, counts):
        before = counts.copy()
        self.k.trsm_right_upper(b, u, counts)
        m, r = b.shape
        assert counts.modular_reductions - before.modular_reductions == (2 * m * r if r else 0)
        assert counts.field_inv - before.field_inv == r
        self.calls += 1


def test_injected_kernels_match_native(pb):
    """pluq(kernels=...) drives the injected strategy and gives the native/oracle result."""
    rng = np.random.default_rng(123)
    for trial in range(12):
        m, n = (int(x) for x in rng.integers(1, 60, 2))
        p = int(rng.choice([3, 101, 65521]))
        a0 = orc.gen_xy_rank(m, n, int(rng.integers(0, min(m, n) + 1)), p, trial) if trial % 2 else rng.integers(0, p, (m, n))
        field = pb.PrimeField(p)
        kern = _Recording(pb, field)
        c1, c2 = pb.OpCounts(), pb.OpCounts()
        a = pb.DenseMatrix(field, a0)
        b = pb.DenseMatrix(field, a0)
        f1 = pb.pluq(a, threshold=2, kernels=kern, counts=c1)
        f2 = pb.pluq(b, threshold=2, counts=c2)
        assert f1.p_perm == f2.p_perm and f1.q_perm == f2.q_perm and f1.rank == f2.rank
        assert np.array_equal(a.data, b.data) and c1 == c2
    assert kern.calls > 0


def test_workspace_scratch_is_bounded(pb):  # test_recursive.py:198-204
    ws = pb.TrackingWorkspace()
    a0 = orc.gen_xy_rank(64, 64, 32, 101, 9)
    a = pb.DenseMatrix(pb.PrimeField(101), a0)
    pb.pluq(a, threshold=8, workspace=ws)
    assert ws.peak_elements <= ws.max_scratch_block + 2 * (64 + 64)
    assert ws.live_elements == 0


# ---------------------------------------------------------------------------------------
# whole-decomposition parity vs the oracle
# ---------------------------------------------------------------------------------------


def _oracle(a0, p, thr=30):
    x = a0.astype(orc.field_dtype(p))
    c = orc.Counts()
    P, Q, r, c = orc.pluq(x, p, thr, c)
    return P, Q, r, x, c.as_tuple()


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes_vs_oracle(pb, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(6):
        m, n = (int(x) for x in rng.integers(1, 400, 2))
        p = int(rng.choice([2, 101, 65521, 8388593]))
        thr = int(rng.choice([1, 4, 30, 30]))
        kind = int(rng.integers(0, 3))
        if kind == 0:
            a0 = rng.integers(0, p, (m, n))
        elif kind == 1:
            a0 = orc.gen_xy_rank(m, n, int(rng.integers(0, min(m, n) + 1)), p, seed)
        else:
            a0 = rng.integers(1, p, (m, n)) * (rng.random((m, n)) < 0.03)
        P, Q, r, packed, cnt = _oracle(a0, p, thr)
        a = pb.DenseMatrix(pb.PrimeField(p), a0)
        c = pb.OpCounts()
        f = pb.pluq(a, threshold=thr, counts=c)
        _check(f, a.data, P, Q, r, packed, cnt, c)


@pytest.mark.parametrize("small_cap", [0, 1, 64 * 64])
def test_driver_paths_agree(pb, small_cap):
    """Force the host recursion to walk smaller nodes (small-node kernel cap) — same bits."""
    from paper_1301_4438_b200 import _native

    ctx = _native.context()
    a0 = orc.gen_xy_rank(300, 260, 180, 65521, 4)
    P, Q, r, packed, cnt = _oracle(a0, 65521)
    ctx.set_option("small_cap", max(small_cap, 1))
    try:
        a = pb.DenseMatrix(pb.PrimeField(65521), a0)
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
    finally:
        ctx.set_option("small_cap", 128 * 128)
    _check(f, a.data, P, Q, r, packed, cnt, c)


def test_large_modulus(pb):
    p = 2147483629  # prime < 2^31
    rng = np.random.default_rng(5)
    a0 = orc.gen_xy_rank(150, 170, 90, p, 3)
    P, Q, r, packed, cnt = _oracle(a0, p)
    a = pb.DenseMatrix(pb.PrimeField(p, allow_large_modulus=True), a0)
    c = pb.OpCounts()
    f = pb.pluq(a, counts=c)
    _check(f, a.data, P, Q, r, packed, cnt, c)


def test_cfg1_full(pb):
    a0 = orc.gen_cfg1(seed=0)
    P, Q, r, packed, cnt = _oracle(a0, 65521)
    a = pb.DenseMatrix(pb.PrimeField(65521), a0)
    c = pb.OpCounts()
    f = pb.pluq(a, counts=c)
    assert r == 384
    _check(f, a.data, P, Q, r, packed, cnt, c)


def test_cfg4_shape_scaled(pb):
    a0, rows, cols = orc.gen_cfg4(seed=2, m=512, n=1024, r=256)
    P, Q, r, packed, cnt = _oracle(a0, 8388593)
    a = pb.DenseMatrix(pb.PrimeField(8388593), a0)
    c = pb.OpCounts()
    f = pb.pluq(a, counts=c)
    _check(f, a.data, P, Q, r, packed, cnt, c)
    assert pb.row_rank_profile(f) == tuple(int(v) for v in rows)
    assert pb.col_rank_profile(f) == tuple(int(v) for v in cols)


def test_cfg5_shape_scaled(pb):
    a0 = orc.gen_xy_rank(1024, 1024, 512, 65521, 5)
    P, Q, r, packed, cnt = _oracle(a0, 65521)
    a = pb.DenseMatrix(pb.PrimeField(65521), a0)
    c = pb.OpCounts()
    f = pb.pluq(a, counts=c)
    _check(f, a.data, P, Q, r, packed, cnt, c)


def test_cfg3_shape_scaled(pb):
    a0 = orc.gen_cfg3(seed=1, n=1536)
    P, Q, r, packed, cnt = _oracle(a0, 65521)
    a = pb.DenseMatrix(pb.PrimeField(65521), a0)
    c = pb.OpCounts()
    f = pb.pluq(a, counts=c)
    _check(f, a.data, P, Q, r, packed, cnt, c)


def test_batched_vs_oracle(pb):
    import torch

    p = 65521
    batch = orc.gen_cfg2(seed=7, batch=256)
    batch[::5] = np.stack([orc.gen_xy_rank(64, 64, 40, p, s) for s in range(0, 256, 5)])
    batch[3] = 0
    t = torch.from_numpy(batch).cuda().to(torch.int32)
    res = pb.pluq_batched(t, p, 30, with_counts=True)
    counts = res.counts.cpu().numpy()
    for b in range(256):
        P, Q, r, packed, cnt = _oracle(batch[b], p)
        assert int(res.ranks[b]) == r
        assert np.array_equal(res.p_sigma[b].cpu().numpy(), P) and np.array_equal(res.q_sigma[b].cpu().numpy(), Q)
        assert np.array_equal(t[b].cpu().numpy(), packed.astype(np.int64))
        assert tuple(int(v) for v in counts[b]) == cnt


def test_batched_host_buffers(pb):
    p = 65521
    batch = orc.gen_cfg2(seed=8, batch=64).astype(np.float64)
    orig = batch.copy()
    res = pb.pluq_batched(batch, p, 30)
    for b in range(0, 64, 7):
        P, Q, r, packed, _ = _oracle(orig[b].astype(np.int64), p)
        assert res.ranks[b] == r and np.array_equal(res.p_sigma[b], P)
        assert np.array_equal(batch[b], packed)


def test_full_scale_cfg3_invariants(pb):
    """cfg3 at its BASELINE size: the oracle is too slow in a test, so check rank,
    packed structure and Freivalds reconstruction on the device."""
    import torch
    from paper_1301_4438_b200 import verify

    n, p = 8192, 65521
    a0 = orc.gen_cfg3(seed=0, n=n)
    orig = torch.from_numpy(a0).cuda().to(torch.int32)
    a = pb.DenseMatrix(pb.PrimeField(p), orig.clone())
    f = pb.pluq(a)
    assert f.rank == n
    assert verify.structure_ok(f)
    assert verify.freivalds(orig, f, probes=2)
    # generic input: P = Q = identity unless a leading minor vanishes (prob ~ n/p)
    bad = verify.freivalds(orig, pb.PluqFactors(f.p_perm, f.q_perm, f.rank,
                                                pb.DenseMatrix(pb.PrimeField(p), (a.data + 1) % p)), probes=1)
    assert not bad


# ---------------------------------------------------------------------------------------
# speculative no-pivot path (generic rank profile) on large nodes
# ---------------------------------------------------------------------------------------

SPEC_CASES = [
    ("full", 200, 200, None, 65521),
    ("full_tall", 300, 120, None, 65521),
    ("full_wide", 120, 300, None, 65521),
    ("xy_rank97", 200, 180, 97, 65521),      # zero pivot mid-block: finish with t > 0
    ("xy_rank64", 192, 192, 64, 65521),      # zero pivot at a block boundary: t = 0
    ("xy_rank5", 150, 170, 5, 1009),
    ("full_p23", 160, 160, None, 8388593),   # 3-limb tensor-core GEMM inside
    ("profile", 200, 240, 60, 8388593),      # non-generic (prescribed profiles): restore + recursion
    ("zero", 130, 140, 0, 101),
]


@pytest.mark.parametrize("name,m,n,r,p", SPEC_CASES)
def test_speculative_path_vs_oracle(pb, name, m, n, r, p):
    from paper_1301_4438_b200 import _native

    rng = np.random.default_rng(m * n + 7)
    if name == "profile":
        a0, _, _ = orc.gen_cfg4(seed=3, m=m, n=n, r=r, p=p)
    elif name == "zero":
        a0 = np.zeros((m, n), dtype=np.int64)
    elif r is None:
        a0 = rng.integers(0, p, (m, n))
    else:
        a0 = orc.gen_xy_rank(m, n, r, p, 11)
    P, Q, R, packed, cnt = _oracle(a0, p)
    ctx = _native.context()
    ctx.set_option("small_cap", 1)       # every node is "large": the speculative path runs
    ctx.set_option("spec_block", 16)
    ctx.set_option("spec_panel", 48)     # several panels with inner blocks
    ctx.set_option("spec_check", 3)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0)
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        st = pb.last_stats()
    finally:
        ctx.set_option("small_cap", 128 * 128)
        ctx.set_option("spec_block", 128)
        ctx.set_option("spec_panel", 1024)
        ctx.set_option("spec_check", 16)
    _check(f, a.data, P, Q, R, packed, cnt, c)
    if name in ("profile",):
        assert st["speculative_fail"] >= 1
    else:
        assert st["speculative_ok"] >= 1


# 128-wide diagonal blocks (diag_lazy_kernel) with zero pivots inside / on the edge of a
# full block and look-ahead between two panels of 256 columns
SPEC128_CASES = [
    ("full", 400, 400, None),
    ("rank200", 400, 380, 200),     # zero pivot at t = 72 of the second 128-block
    ("rank128", 384, 384, 128),     # zero pivot on a block boundary
    ("rank50", 300, 300, 50),       # zero pivot inside the first block
    ("rank300", 600, 640, 300),     # zero pivot in the SECOND panel: the look-ahead side update
                                    # of panel 0 (snapshot taken before the stop) must complete
    ("profile", 300, 400, 150),     # non-generic: restore + exact recursion
]


@pytest.mark.parametrize("name,m,n,r", SPEC128_CASES)
def test_speculative_128_blocks_vs_oracle(pb, name, m, n, r):
    from paper_1301_4438_b200 import _native

    p = 65521
    if name == "profile":
        a0, _, _ = orc.gen_cfg4(seed=5, m=m, n=n, r=r, p=p)
    elif r is None:
        a0 = np.random.default_rng(m + n).integers(0, p, (m, n))
    else:
        a0 = orc.gen_xy_rank(m, n, r, p, 13)
    P, Q, R, packed, cnt = _oracle(a0, p)
    ctx = _native.context()
    ctx.set_option("small_cap", 1)
    ctx.set_option("spec_panel", 256)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0)
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        st = pb.last_stats()
    finally:
        ctx.set_option("small_cap", 128 * 128)
        ctx.set_option("spec_panel", 1024)
    _check(f, a.data, P, Q, R, packed, cnt, c)
    assert st["speculative_fail" if name == "profile" else "speculative_ok"] >= 1


@pytest.mark.parametrize("bsz", [1, 5, 17, 100])
def test_batched_host_odd_sizes(pb, bsz):
    """Host-buffer batches whose tent-shaped chunking leaves empty / uneven chunks."""
    p = 65521
    rng = np.random.default_rng(bsz)
    batch = rng.integers(0, p, (bsz, 64, 64)).astype(np.float64)
    batch[::3] = np.stack([orc.gen_xy_rank(64, 64, 20, p, s).astype(np.float64) for s in range(0, bsz, 3)])
    orig = batch.copy()
    res = pb.pluq_batched(batch, p, 30)
    for b in range(bsz):
        P, Q, r, packed, _ = _oracle(orig[b].astype(np.int64), p)
        assert res.ranks[b] == r and np.array_equal(res.p_sigma[b], P) and np.array_equal(res.q_sigma[b], Q)
        assert np.array_equal(batch[b], packed)
