"""The rank-profile route for non-generic blocks (csrc/pluq_rpm.cuh).

The kernel finishes a block that is not generic without replaying the reference
recursion in field arithmetic.  It relies on two facts about Algorithm 1
(recursive.py:186-256 with the Algorithm 2 base case, iterative.py:23-91):

  (1) P, Q, rank and OpCounts of pluq(A) equal those of pluq(R_A), R_A being the rank
      profile matrix, and they are reproduced by replaying the recursion symbolically
      on R_A's pattern (index lists only);
  (2) the packed output of pluq(A) is the unpivoted LU of A[P^-1][:, Q].

The CPU tests pin both facts and a Python model of the kernel's three phases against
the oracle and the reference goldens; the GPU tests pin the kernel itself.
"""

import numpy as np
import pytest

from oracle import pluq_oracle as orc

# --------------------------------------------------------------------------------------
# Python model of the kernel (pluq_rpm.cuh): rpm_rows, sym_base, sym_rec
# --------------------------------------------------------------------------------------


def rpm_rows(a, p):
    """Row-order elimination -> rp[i] = column of row i's pivot in R_A (or -1)."""
    w = np.asarray(a, dtype=np.int64) % p
    m, n = w.shape
    rp = [-1] * m
    for i in range(m):
        nz = np.flatnonzero(w[i])
        if nz.size == 0:
            continue
        j = int(nz[0])
        rp[i] = j
        piv = int(w[i, j])
        for k in range(i + 1, m):
            f = int(w[k, j])
            if f:
                w[k] = (piv * w[k] - f * w[i]) % p
    return rp


class _Cnt:
    def __init__(self):
        self.mul = self.add = self.inv = self.red = 0

    def tuple(self):
        return (self.mul, self.add, self.inv, self.red)


def _mm(c, m, n, k):
    if m and n and k:
        c.red += m * n
        c.mul += m * n * k
        c.add += m * n * k


def _tl(c, r, n):
    if r and n:
        c.red += r * n
        c.mul += n * (r * (r - 1) // 2)
        c.add += n * (r * (r - 1) // 2)


def _tu(c, m, r):
    if r:
        c.inv += r
        if m:
            c.red += 2 * m * r
            c.mul += m * (r * (r + 1) // 2)
            c.add += m * (r * (r - 1) // 2)


def sym_base(rows, cols, rp, cnt):
    m, n = len(rows), len(cols)
    cpos = {c: b for b, c in enumerate(cols)}
    lr = [cpos.get(rp[r], -1) if rp[r] >= 0 else -1 for r in rows]
    lc = [-1] * n
    for a, b in enumerate(lr):
        if b >= 0:
            lc[b] = a
    ro, co = [], []
    i = j = 0
    while i < m or j < n:
        piv = None
        if j < n and 0 <= lc[j] < i:
            piv = (lc[j], j)
            j += 1
        if piv is None and i < m:
            if 0 <= lr[i] < j:
                piv = (i, lr[i])
                i += 1
            elif j < n and lr[i] == j:
                piv = (i, j)
                i += 1
                j += 1
        if piv is None:
            i, j = min(i + 1, m), min(j + 1, n)
            continue
        ro.append(piv[0])
        co.append(piv[1])
    for k, (pr, pc) in enumerate(zip(ro, co)):
        below = m - 1 - pr - sum(1 for t in range(k) if ro[t] > pr)
        right = n - 1 - pc - sum(1 for t in range(k) if co[t] > pc)
        if below > 0:
            cnt.inv += 1
            cnt.mul += below + below * right
            cnt.add += below * right
            cnt.red += below + below * right
    rowat = ro + [x for x in range(m) if x not in set(ro)]
    colat = co + [x for x in range(n) if x not in set(co)]
    return orc.perm_inverse(np.array(rowat, dtype=np.int64)), np.array(colat, dtype=np.int64), len(ro)


def sym_rec(rows, cols, rp, thr, cnt):
    m, n = len(rows), len(cols)
    if m == 0 or n == 0:
        return orc._ident(m), orc._ident(n), 0
    if m == 1 or n == 1 or min(m, n) <= thr:
        return sym_base(rows, cols, rp, cnt)
    kr, kc = m // 2, n // 2
    p1, q1, r1 = sym_rec(rows[:kr], cols[:kc], rp, thr, cnt)
    ip1 = orc.perm_inverse(p1)
    rt = [rows[ip1[t]] for t in range(kr)]
    cl = [cols[q1[t]] for t in range(kc)]
    _tl(cnt, r1, n - kc); _tu(cnt, m - kr, r1)
    _mm(cnt, kr - r1, n - kc, r1); _mm(cnt, m - kr, kc - r1, r1); _mm(cnt, m - kr, n - kc, r1)
    p2, q2, r2 = sym_rec(rt[r1:], cols[kc:], rp, thr, cnt)
    p3, q3, r3 = sym_rec(rows[kr:], cl[r1:], rp, thr, cnt)
    ip3 = orc.perm_inverse(p3)
    hr = [rows[kr + ip3[t]] for t in range(m - kr)]
    hc = [cols[kc + q2[t]] for t in range(n - kc)]
    m4, n4 = m - kr - r3, n - kc - r2
    _tu(cnt, r3, r2); _tl(cnt, r3, r2); _tu(cnt, m4, r2); _tl(cnt, r3, n4)
    _mm(cnt, r3, n4, r2); _mm(cnt, m4, n4, r2); _mm(cnt, m4, n4, r3)
    p4, q4, r4 = sym_rec(hr[r3:], hc[r2:], rp, thr, cnt)
    s = orc.s_perm(r1, r2, r3, r4, kr, m)
    t = orc.t_perm(r1, r2, r3, r4, kc, n)
    pl = orc.perm_compose(p1, orc.perm_block_diag([orc._ident(r1), p2]))
    pr_ = orc.perm_compose(p3, orc.perm_block_diag([orc._ident(r3), p4]))
    pp = orc.perm_compose(orc.perm_block_diag([pl, pr_]), s)
    ql = orc.perm_compose(orc.perm_block_diag([orc._ident(r1), q3]), q1)
    qr = orc.perm_compose(orc.perm_block_diag([orc._ident(r2), q4]), q2)
    return pp, orc.perm_compose(t, orc.perm_block_diag([ql, qr])), r1 + r2 + r3 + r4


def model_pluq(a, p, thr):
    """The kernel's route end to end: R_A, symbolic Alg.1, unpivoted LU of A[P^-1][:, Q]."""
    m, n = a.shape
    rp = rpm_rows(a, p)
    cnt = _Cnt()
    P, Q, r = sym_rec(list(range(m)), list(range(n)), rp, thr, cnt)
    ap = np.asarray(a, dtype=np.int64)[orc.perm_inverse(P)][:, Q].astype(orc.field_dtype(p))
    P2, Q2, r2, _ = orc.pluq(ap, p, 10**9)  # Alg.2 with no pivoting needed == unpivoted LU
    assert r2 == r and np.array_equal(P2, orc._ident(m)) and np.array_equal(Q2, orc._ident(n))
    return P, Q, r, ap, cnt.tuple()


def _rand_nongeneric(rng, p, m, n):
    kind = rng.integers(0, 3)
    if kind == 0:
        return rng.integers(0, p, (m, n))
    if kind == 1:
        r = int(rng.integers(0, min(m, n) + 1))
        return (rng.integers(0, p, (m, r)) @ rng.integers(0, p, (r, n))) % p
    return rng.integers(0, p, (m, n)) * (rng.random((m, n)) < 0.12)


# --------------------------------------------------------------------------------------
# CPU: the model against the oracle and the reference's own goldens
# --------------------------------------------------------------------------------------


def test_model_matches_oracle_random():
    rng = np.random.default_rng(2024)
    for _ in range(250):
        p = int(rng.choice([2, 3, 5, 7, 11, 101, 65521]))
        m, n = int(rng.integers(1, 48)), int(rng.integers(1, 48))
        thr = int(rng.choice([1, 2, 3, 5, 8, 30]))
        a = _rand_nongeneric(rng, p, m, n)
        x = a.astype(orc.field_dtype(p))
        P, Q, r, cnt = orc.pluq(x, p, thr)
        mP, mQ, mr, mpacked, mcnt = model_pluq(a, p, thr)
        assert r == mr and np.array_equal(P, mP) and np.array_equal(Q, mQ), (p, m, n, thr)
        assert np.array_equal(x, mpacked), (p, m, n, thr)
        assert (cnt.field_mul, cnt.field_add, cnt.field_inv, cnt.modular_reductions) == mcnt


def test_model_matches_reference_goldens(golden):
    z, man = golden
    seen = 0
    for e in man:
        if e["route"] != "recursive" or e["m"] * e["n"] > 4096 or e["m"] * e["n"] == 0:
            continue
        a = z[e["key"] + "_in"]
        P, Q, r, packed, cnt = model_pluq(a, e["p"], e["threshold"])
        assert r == e["rank"]
        assert np.array_equal(P, z[e["key"] + "_P"]) and np.array_equal(Q, z[e["key"] + "_Q"])
        assert list(cnt) == e["counts"]
        seen += 1
    assert seen > 50


def test_rank_profile_matrix_is_the_invariant():
    """pluq(A) and pluq(R_A) agree on P, Q, rank and OpCounts."""
    rng = np.random.default_rng(5)
    for _ in range(150):
        p = int(rng.choice([2, 3, 7, 65521]))
        m, n = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        thr = int(rng.choice([1, 3, 8, 30]))
        a = _rand_nongeneric(rng, p, m, n).astype(orc.field_dtype(p))
        P, Q, r, c = orc.pluq(a.copy(), p, thr)
        R = np.zeros_like(a)
        for i, j in orc.support_pairs(P, Q, r):
            R[i, j] = 1
        P2, Q2, r2, c2 = orc.pluq(R, p, thr)
        assert r == r2 and np.array_equal(P, P2) and np.array_equal(Q, Q2)
        assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == \
               (c2.field_mul, c2.field_add, c2.field_inv, c2.modular_reductions)


# --------------------------------------------------------------------------------------
# GPU: the kernel
# --------------------------------------------------------------------------------------


@pytest.fixture
def ctx(cuda_ok):
    from paper_1301_4438_b200 import _native

    c = _native.context()
    yield c
    c.set_option("exact_kernel", 1)
    c.set_option("try_generic", 1)
    c.set_option("rpm_threads", 512)


RPM_CASES = [  # (p, m, n, threshold, batch)
    (2, 64, 64, 30, 48), (3, 64, 64, 30, 48), (7, 64, 64, 4, 32), (65521, 64, 64, 30, 32),
    (5, 17, 40, 3, 40), (11, 48, 33, 1, 32), (2, 1, 64, 30, 16), (3, 64, 1, 30, 16),
    (101, 31, 31, 30, 24), (2, 96, 80, 16, 12), (8388593, 40, 40, 7, 16), (67108859, 33, 20, 5, 16),
]


def _batch(rng, p, m, n, b):
    return np.stack([_rand_nongeneric(rng, p, m, n) for _ in range(b)]).astype(np.int64)


@pytest.mark.gpu
@pytest.mark.parametrize("try_generic", [1, 0])
@pytest.mark.parametrize("case", RPM_CASES)
def test_rpm_kernel_batched(ctx, case, try_generic):
    import torch

    import paper_1301_4438_b200 as pb

    p, m, n, thr, b = case
    ctx.set_option("try_generic", try_generic)
    ctx.set_option("exact_kernel", 1)
    rng = np.random.default_rng(p + m * 7 + n * 13 + thr)
    batch = _batch(rng, p, m, n, b)
    t = torch.from_numpy(batch).cuda().to(torch.int32)
    res = pb.pluq_batched(t, p, thr, with_counts=True)
    out = t.cpu().numpy()
    counts = res.counts.cpu().numpy()
    for k in range(b):
        x = batch[k].astype(orc.field_dtype(p))
        P, Q, r, c = orc.pluq(x, p, thr)
        assert int(res.ranks[k]) == r, k
        assert np.array_equal(res.p_sigma[k].cpu().numpy(), P), k
        assert np.array_equal(res.q_sigma[k].cpu().numpy(), Q), k
        assert np.array_equal(out[k], x.astype(np.int64)), k
        assert tuple(int(v) for v in counts[k]) == (c.field_mul, c.field_add, c.field_inv, c.modular_reductions)


@pytest.mark.gpu
@pytest.mark.parametrize("threads", [64, 128, 256, 512])
def test_rpm_kernel_block_sizes(ctx, threads):
    import torch

    import paper_1301_4438_b200 as pb

    p, m, n, thr = 3, 64, 64, 30
    ctx.set_option("try_generic", 0)
    ctx.set_option("rpm_threads", threads)
    batch = _batch(np.random.default_rng(threads), p, m, n, 24)
    t = torch.from_numpy(batch).cuda().to(torch.int32)
    res = pb.pluq_batched(t, p, thr)
    out = t.cpu().numpy()
    for k in range(24):
        x = batch[k].astype(orc.field_dtype(p))
        P, Q, r, _ = orc.pluq(x, p, thr)
        assert int(res.ranks[k]) == r and np.array_equal(res.p_sigma[k].cpu().numpy(), P)
        assert np.array_equal(out[k], x.astype(np.int64))


@pytest.mark.gpu
def test_rpm_single_small_matrices(ctx):
    """pluq() on small non-generic matrices (one CTA leaf) through the rank-profile kernel."""
    import paper_1301_4438_b200 as pb

    rng = np.random.default_rng(77)
    for trial in range(40):
        p = int(rng.choice([2, 3, 7, 65521]))
        m, n = int(rng.integers(1, 128)), int(rng.integers(1, 128))
        thr = int(rng.choice([1, 5, 30]))
        a0 = _rand_nongeneric(rng, p, m, n)
        x = a0.astype(orc.field_dtype(p))
        P, Q, r, c = orc.pluq(x, p, thr)
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(orc.field_dtype(p)))
        cc = pb.OpCounts()
        f = pb.pluq(a, threshold=thr, counts=cc)
        assert f.rank == r and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
        assert np.array_equal(np.asarray(a.data, dtype=np.int64), x.astype(np.int64))
        assert [cc.field_mul, cc.field_add, cc.field_inv, cc.modular_reductions] == \
               [c.field_mul, c.field_add, c.field_inv, c.modular_reductions]
