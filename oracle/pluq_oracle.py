"""CPU restatement of the reference PLUQ-mod-p path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line whose behaviour it restates.
Arrays are numpy, storage dtype follows the reference field rule
(`field.py:75-81`): float64 when (p-1)^2 * 8192 <= 2^53, else int64.

Results that must be bit-identical to the reference: the packed matrix,
P.sigma, Q.sigma, rank and the four OpCounts tallies.  The elimination
kernels (mm_acc / trsm) compute exact modular results, so any exact
evaluation order gives identical bits; only the recursion shape (split at
(m//2, n//2), m==1/n==1 before threshold, threshold test) and the base-case
pivot search order decide P and Q, and those are restated literally.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "Counts",
    "field_dtype",
    "max_accumulate",
    "inverse_mod",
    "matmul_mod",
    "mm_acc",
    "trsm_left_unit_lower",
    "trsm_right_upper",
    "basecase",
    "pluq",
    "pluq_iterative",
    "support_pairs",
    "row_rank_profile",
    "col_rank_profile",
    "leading_rank_profiles",
    "reconstruct",
    "perm_compose",
    "perm_inverse",
    "perm_block_diag",
    "s_perm",
    "t_perm",
    "gen_cfg1",
    "gen_cfg2",
    "gen_cfg3",
    "gen_cfg4",
    "gen_cfg5",
    "gen_xy_rank",
    "effective_work",
    "pluq_batch",
]

_F64_EXACT = 1 << 53
_I64_EXACT = (1 << 63) - 1


@dataclass
class Counts:
    """Mirror of OpCounts (`matrix.py:22-43`)."""

    field_mul: int = 0
    field_add: int = 0
    field_inv: int = 0
    modular_reductions: int = 0

    def as_tuple(self):
        return (self.field_mul, self.field_add, self.field_inv, self.modular_reductions)


# --------------------------------------------------------------------------------------
# field arithmetic  (field.py:41-52, 65-81, 149-161)
# --------------------------------------------------------------------------------------


def field_dtype(p: int):
    """Storage dtype rule of `PrimeField.__init__` (field.py:75-81)."""
    return np.float64 if (p - 1) ** 2 * 8192 <= _F64_EXACT else np.int64


def max_accumulate(p: int) -> int:
    """Delayed-reduction chunk of `PrimeField.__init__` (field.py:76-81)."""
    sq = (p - 1) ** 2
    if field_dtype(p) is np.float64:
        return max(1, _F64_EXACT // sq - 1) if sq else _F64_EXACT
    return max(1, _I64_EXACT // sq - 1) if sq else _I64_EXACT


def inverse_mod(a: int, p: int) -> int:
    """Extended Euclid inverse (field.py:41-52); ZeroDivisionError on 0."""
    a %= p
    if a == 0:
        raise ZeroDivisionError("inverse of 0")
    return pow(int(a), -1, int(p))


def matmul_mod(a: np.ndarray, b: np.ndarray, p: int) -> np.ndarray:
    """Exact (a @ b) mod p with K chunked at the overflow-safe bound (field.py:149-161)."""
    dt = field_dtype(p)
    m, k = a.shape
    n = b.shape[1]
    out = np.zeros((m, n), dtype=dt)
    if k == 0:
        return out
    step = max_accumulate(p)
    for lo in range(0, k, step):
        out += a[:, lo:lo + step].astype(dt, copy=False) @ b[lo:lo + step].astype(dt, copy=False)
        np.mod(out, p, out=out)
    return out


# --------------------------------------------------------------------------------------
# kernels  (kernels.py:38-120) — exact results + the reference's closed-form charges
# --------------------------------------------------------------------------------------


def mm_acc(c, a, b, p, counts: Counts) -> None:
    """C <- C - A B mod p (kernels.py:38-55); charges m*n reductions, m*n*k mul/add."""
    m, k = a.shape
    k2, n = b.shape
    if c.shape != (m, n) or k2 != k:
        raise ValueError(f"mm_acc shapes C{c.shape} A{a.shape} B{b.shape}")
    if k == 0 or m == 0 or n == 0:
        return
    counts.modular_reductions += m * n
    counts.field_mul += m * n * k
    counts.field_add += m * n * k
    c[...] = np.mod(c - matmul_mod(a, b, p), p)


def trsm_left_unit_lower(l, b, p, counts: Counts) -> None:
    """B <- L^-1 B, L unit lower, diagonal implicit (kernels.py:59-83)."""
    r = l.shape[0]
    if l.shape[1] != r or b.shape[0] != r:
        raise ValueError(f"trsm shapes L{l.shape} B{b.shape}")
    n = b.shape[1]
    if r == 0 or n == 0:
        return
    counts.modular_reductions += r * n
    counts.field_mul += n * (r * (r - 1) // 2)
    counts.field_add += n * (r * (r - 1) // 2)
    _fwd(l, b, p)


def _fwd(l, b, p):
    # blocked forward substitution; exact, so any blocking gives the same bits
    r = l.shape[0]
    if r <= 32:
        for i in range(1, r):
            b[i] = np.mod(b[i] - matmul_mod(l[i:i + 1, :i], b[:i], p)[0], p)
        return
    h = r // 2
    _fwd(l[:h, :h], b[:h], p)
    b[h:] = np.mod(b[h:] - matmul_mod(l[h:, :h], b[:h], p), p)
    _fwd(l[h:, h:], b[h:], p)


def trsm_right_upper(b, u, p, counts: Counts) -> None:
    """B <- B U^-1, U upper with nonzero diagonal (kernels.py:85-120)."""
    r = u.shape[0]
    if u.shape[1] != r or b.shape[1] != r:
        raise ValueError(f"trsm shapes B{b.shape} U{u.shape}")
    m = b.shape[0]
    if r == 0:
        return
    diag = np.array([u[t, t] for t in range(r)])
    if np.any(diag == 0):
        raise ZeroDivisionError("upper triangular factor has a zero diagonal entry")
    counts.field_inv += r
    if m == 0:
        return
    counts.modular_reductions += 2 * m * r
    counts.field_mul += m * (r * (r + 1) // 2)
    counts.field_add += m * (r * (r - 1) // 2)
    inv = np.array([inverse_mod(int(d), p) for d in diag], dtype=b.dtype)
    _bwd(b, u, inv, p)


def _bwd(b, u, inv, p):
    r = u.shape[0]
    if r <= 32:
        for j in range(r):
            col = b[:, j]
            if j:
                col = np.mod(col - matmul_mod(b[:, :j], u[:j, j:j + 1], p)[:, 0], p)
            b[:, j] = np.mod(col * inv[j], p)
        return
    h = r // 2
    _bwd(b[:, :h], u[:h, :h], inv[:h], p)
    b[:, h:] = np.mod(b[:, h:] - matmul_mod(b[:, :h], u[:h, h:], p), p)
    _bwd(b[:, h:], u[h:, h:], inv[h:], p)


# --------------------------------------------------------------------------------------
# permutation algebra  (matrix.py:161-246, recursive.py:77-99)
# sigma convention: Mat(sigma)[i, sigma(i)] = 1  (matrix.py:3-11)
# --------------------------------------------------------------------------------------


def perm_compose(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """sigma of Mat(a) @ Mat(b) (matrix.py:201-205)."""
    return b[a]


def perm_inverse(a: np.ndarray) -> np.ndarray:
    inv = np.empty_like(a)
    inv[a] = np.arange(a.shape[0], dtype=a.dtype)
    return inv


def perm_block_diag(parts) -> np.ndarray:
    """Diag(p1, ..., pk) (matrix.py:238-246)."""
    out, off = [], 0
    for s in parts:
        out.append(np.asarray(s, dtype=np.int64) + off)
        off += len(s)
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


def _ident(s: int) -> np.ndarray:
    return np.arange(s, dtype=np.int64)


def s_perm(r1, r2, r3, r4, k, m) -> np.ndarray:
    """Row block permutation S (recursive.py:77-85): blocks (1,2,3,4) -> (1,3,2,4)."""
    if not (0 <= r1 + r2 <= k <= m and 0 <= r3 + r4 <= m - k):
        raise ValueError("inconsistent row block sizes")
    a, b = r1 + r2, k - (r1 + r2)
    c = r3 + r4
    sig = _ident(m)
    sig[a:k] = np.arange(a, k) + c
    sig[k:k + c] = np.arange(k, k + c) - b
    return sig


def t_perm(r1, r2, r3, r4, k, n) -> np.ndarray:
    """Column block permutation T (recursive.py:88-99)."""
    if not (0 <= r1 + r3 <= k <= n and 0 <= r2 + r4 <= n - k):
        raise ValueError("inconsistent column block sizes")
    # target order of the source blocks (r1 | r3 | k-r1-r3 | r2 | r4 | rest)
    src_blocks = [(0, r1), (r1, r3), (r1 + r3, k - r1 - r3), (k, r2), (k + r2, r4), (k + r2 + r4, n - k - r2 - r4)]
    order = [0, 3, 1, 4, 2, 5]
    # sigma[j] = source column landing at position j of A T^T  (test_recursive.py:137-141)
    sig = np.concatenate([np.arange(src_blocks[o][0], src_blocks[o][0] + src_blocks[o][1]) for o in order])
    # A Mat(T)^T column j is column sigma_T(j) of A  -> sigma_T = sig
    return sig.astype(np.int64)


def _gather_rows(x, g):
    """apply_rows(x, perm) with perm.sigma = g (matrix.py:272-276): new[i] = old[g[i]]."""
    if x.shape[0] and not np.array_equal(g, np.arange(len(g))):
        x[...] = x[g, :]


def _gather_cols(x, g):
    """new[:, j] = old[:, g[j]] (apply_cols(x, perm) uses g = perm.inverse().sigma, matrix.py:279-283)."""
    if x.shape[1] and not np.array_equal(g, np.arange(len(g))):
        x[...] = x[:, g]


# --------------------------------------------------------------------------------------
# base case: Algorithm 2, Z-curve iterative elimination  (iterative.py:30-93)
# Restated with LAZY row/column rotations: arithmetic happens in the original
# coordinates and one gather at the end realises all rotations at once.
# Equivalence: the rotations keep non-pivot rows/cols in original relative
# order, so "rows after the pivot in the current layout" are exactly the
# non-pivot rows with larger original index, and current row i / column j on
# the frontier are still the untouched original row i / column j.
# --------------------------------------------------------------------------------------


def basecase(a: np.ndarray, p: int, counts: Counts, trace=None):
    m, n = a.shape
    piv_row = np.zeros(m, dtype=bool)
    piv_col = np.zeros(n, dtype=bool)
    row_order, col_order = [], []
    r = i = j = 0
    while i < m or j < n:
        if trace is not None:
            trace.append((i, j, r))
        pivot = None
        if j < n:  # column segment A[r:i, j]  (iterative.py:40-44)
            cand = np.flatnonzero((a[:i, j] != 0) & ~piv_row[:i])
            if cand.size:
                pivot = (int(cand[0]), j)
                j += 1
        if pivot is None and i < m:  # row segment A[i, r:j], then corner (iterative.py:45-53)
            cand = np.flatnonzero((a[i, :j] != 0) & ~piv_col[:j])
            if cand.size:
                pivot = (i, int(cand[0]))
                i += 1
            elif j < n and a[i, j] != 0:
                pivot = (i, j)
                i += 1
                j += 1
        if pivot is None:  # (iterative.py:54-57)
            i = min(i + 1, m)
            j = min(j + 1, n)
            continue
        pr, pc = pivot
        below = np.flatnonzero(~piv_row)
        below = below[below > pr]
        right = np.flatnonzero(~piv_col)
        right = right[right > pc]
        if below.size:  # (iterative.py:59-75)
            inv = inverse_mod(int(a[pr, pc]), p)
            counts.field_inv += 1
            mult = np.mod(a[below, pc] * inv, p)
            a[below, pc] = mult
            counts.field_mul += below.size
            counts.modular_reductions += below.size
            if right.size:
                blk = a[np.ix_(below, right)]
                blk = np.mod(blk - np.outer(mult, a[pr, right]), p)
                a[np.ix_(below, right)] = blk
                counts.field_mul += below.size * right.size
                counts.field_add += below.size * right.size
                counts.modular_reductions += below.size * right.size
        piv_row[pr] = True
        piv_col[pc] = True
        row_order.append(pr)
        col_order.append(pc)
        r += 1
    row_at = np.array(row_order + [x for x in range(m) if not piv_row[x]], dtype=np.int64)
    col_at = np.array(col_order + [x for x in range(n) if not piv_col[x]], dtype=np.int64)
    _gather_rows(a, row_at)
    _gather_cols(a, col_at)
    # P.sigma[orig] = final position of orig row; Q.sigma[t] = orig col at t (iterative.py:82-91)
    return perm_inverse(row_at), col_at, r


# --------------------------------------------------------------------------------------
# Algorithm 1 recursion  (recursive.py:159-256)
# --------------------------------------------------------------------------------------


def _rec(x, p, threshold, counts):
    m, n = x.shape
    if m == 0 or n == 0:  # (recursive.py:188-189)
        return _ident(m), _ident(n), 0
    if m == 1 or n == 1 or min(m, n) <= threshold:
        # m==1 / n==1 terminal cases are bit-identical to Alg. 2 on a line
        # (recursive.py:190-193, pinned by test_recursive.py:90-104)
        return basecase(x, p, counts)
    kr, kc = m // 2, n // 2

    p1, q1, r1 = _rec(x[:kr, :kc], p, threshold, counts)
    _gather_rows(x[:kr, kc:], perm_inverse(p1))     # B <- P1^T B
    _gather_cols(x[kr:, :kc], q1)                    # C <- C Q1^T
    trsm_left_unit_lower(x[:r1, :r1], x[:r1, kc:], p, counts)          # D
    trsm_right_upper(x[kr:, :r1], x[:r1, :r1], p, counts)              # E
    mm_acc(x[r1:kr, kc:], x[r1:kr, :r1], x[:r1, kc:], p, counts)       # F
    mm_acc(x[kr:, r1:kc], x[kr:, :r1], x[:r1, r1:kc], p, counts)       # G
    mm_acc(x[kr:, kc:], x[kr:, :r1], x[:r1, kc:], p, counts)           # H

    p2, q2, r2 = _rec(x[r1:kr, kc:], p, threshold, counts)
    p3, q3, r3 = _rec(x[kr:, r1:kc], p, threshold, counts)

    ip3, ip2 = perm_inverse(p3), perm_inverse(p2)
    _gather_rows(x[kr:, kc:], ip3)
    _gather_cols(x[kr:, kc:], q2)
    _gather_rows(x[kr:, :r1], ip3)
    _gather_rows(x[r1:kr, :r1], ip2)
    _gather_cols(x[:r1, kc:], q2)
    _gather_cols(x[:r1, r1:kc], q3)

    u2 = x[r1:r1 + r2, kc:kc + r2]
    l3 = x[kr:kr + r3, r1:r1 + r3]
    trsm_right_upper(x[kr:kr + r3, kc:kc + r2], u2, p, counts)          # I
    scratch = x[kr:kr + r3, kc:kc + r2].copy()
    trsm_left_unit_lower(l3, scratch, p, counts)                        # J (scratch)
    trsm_right_upper(x[kr + r3:, kc:kc + r2], u2, p, counts)            # K
    trsm_left_unit_lower(l3, x[kr:kr + r3, kc + r2:], p, counts)        # N
    mm_acc(x[kr:kr + r3, kc + r2:], scratch, x[r1:r1 + r2, kc + r2:], p, counts)            # O
    mm_acc(x[kr + r3:, kc + r2:], x[kr + r3:, kc:kc + r2], x[r1:r1 + r2, kc + r2:], p, counts)
    mm_acc(x[kr + r3:, kc + r2:], x[kr + r3:, r1:r1 + r3], x[kr:kr + r3, kc + r2:], p, counts)

    p4, q4, r4 = _rec(x[kr + r3:, kc + r2:], p, threshold, counts)

    _gather_rows(x[kr + r3:, :kc + r2], perm_inverse(p4))
    _gather_cols(x[:kr + r3, kc + r2:], q4)

    s = s_perm(r1, r2, r3, r4, kr, m)
    t = t_perm(r1, r2, r3, r4, kc, n)
    _gather_rows(x, perm_inverse(s))
    _gather_cols(x, t)

    # P = Diag(P1 Diag(I,P2), P3 Diag(I,P4)) S ; Q = T Diag(Diag(I,Q3) Q1, Diag(I,Q4) Q2)
    pl = perm_compose(p1, perm_block_diag([_ident(r1), p2]))
    pr_ = perm_compose(p3, perm_block_diag([_ident(r3), p4]))
    pp = perm_compose(perm_block_diag([pl, pr_]), s)
    ql = perm_compose(perm_block_diag([_ident(r1), q3]), q1)
    qr = perm_compose(perm_block_diag([_ident(r2), q4]), q2)
    qq = perm_compose(t, perm_block_diag([ql, qr]))
    return pp, qq, r1 + r2 + r3 + r4


def pluq(a: np.ndarray, p: int, threshold: int = 30, counts: Counts | None = None):
    """In-place PLUQ of `a` (field dtype array). Returns (P.sigma, Q.sigma, r, counts)."""
    if threshold < 1:
        raise ValueError("threshold must be a positive integer")
    counts = counts if counts is not None else Counts()
    pp, qq, r = _rec(a, p, threshold, counts)
    return pp, qq, r, counts


def pluq_iterative(a: np.ndarray, p: int, counts: Counts | None = None):
    """Alg. 2 on the whole matrix (iterative.py:23-27)."""
    counts = counts if counts is not None else Counts()
    pp, qq, r = basecase(a, p, counts)
    return pp, qq, r, counts


# --------------------------------------------------------------------------------------
# rank profiles (rank_profile.py:17-35, matrix.py:322-326) and reconstruction (:328-335)
# --------------------------------------------------------------------------------------


def support_pairs(psig, qsig, r):
    inv_p = perm_inverse(np.asarray(psig))
    return [(int(inv_p[t]), int(qsig[t])) for t in range(r)]


def row_rank_profile(psig, qsig, r):
    return tuple(sorted(a for a, _ in support_pairs(psig, qsig, r)))


def col_rank_profile(psig, qsig, r):
    return tuple(sorted(b for _, b in support_pairs(psig, qsig, r)))


def leading_rank_profiles(psig, qsig, r, k, t):
    inside = [(a, b) for a, b in support_pairs(psig, qsig, r) if a < k and b < t]
    return tuple(sorted(a for a, _ in inside)), tuple(sorted(b for _, b in inside))


def reconstruct(packed, psig, qsig, r, p):
    """Mat(P) [L;M] [U V] Mat(Q) mod p (matrix.py:308-335)."""
    m, n = packed.shape
    lm = np.tril(packed[:, :r], -1).astype(np.int64)
    lm[np.arange(r), np.arange(r)] = 1
    uv = packed[:r, :].astype(np.int64).copy()
    uv[:, :r] = np.triu(uv[:, :r])
    prod = matmul_mod(lm, uv, p).astype(np.int64)
    prod = prod[np.asarray(psig), :]
    prod = prod[:, perm_inverse(np.asarray(qsig))]
    return prod


# --------------------------------------------------------------------------------------
# BASELINE.json config generators (SURVEY.md §8(d) draw order), int64 in [0, p)
# --------------------------------------------------------------------------------------


def _mulmod_exact(x: np.ndarray, y: np.ndarray, p: int) -> np.ndarray:
    """Exact X Y mod p for int64 residues (p < 2^32) using float64 BLAS on 16-bit halves."""
    k = x.shape[1]
    if (p - 1) ** 2 * k < _F64_EXACT:
        return np.mod(x.astype(np.float64) @ y.astype(np.float64), p).astype(np.int64)
    assert k < (1 << 21), "16-bit split exact only for K < 2^21"
    x = np.asarray(x, dtype=np.int64)
    y = np.asarray(y, dtype=np.int64)
    x0, x1 = (x & 0xFFFF).astype(np.float64), (x >> 16).astype(np.float64)
    y0, y1 = (y & 0xFFFF).astype(np.float64), (y >> 16).astype(np.float64)

    def mm(u, v):
        return np.mod(u @ v, p).astype(np.int64)

    ll, lh, hl, hh = mm(x0, y0), mm(x0, y1), mm(x1, y0), mm(x1, y1)
    s16, s32 = (1 << 16) % p, (1 << 32) % p
    mid = np.mod(lh + hl, p) * s16 % p
    return (ll + mid + hh * s32 % p) % p


def gen_xy_rank(m, n, r, p, seed, permute=True):
    """cfg1/cfg5 family: A = X Y mod p, X m x r, Y r x n uniform, then row/col perms."""
    rng = np.random.default_rng(seed)
    x = rng.integers(0, p, (m, r), dtype=np.int64)
    y = rng.integers(0, p, (r, n), dtype=np.int64)
    a = _mulmod_exact(x, y, p)
    if permute:
        a = a[rng.permutation(m)][:, rng.permutation(n)]
    return np.ascontiguousarray(a)


def gen_cfg1(seed=0, m=512, n=512, r=384, p=65521):
    return gen_xy_rank(m, n, r, p, seed)


def gen_cfg2(seed=0, batch=4096, m=64, n=64, p=65521):
    rng = np.random.default_rng(seed)
    return rng.integers(0, p, (batch, m, n), dtype=np.int64)


def gen_cfg3(seed=0, n=8192, p=65521):
    rng = np.random.default_rng(seed)
    return rng.integers(0, p, (n, n), dtype=np.int64)


def gen_cfg4(seed=0, m=16384, n=32768, r=8192, p=8388593):
    """Prescribed rank profiles (I, J): A = X Y with echelon-forced X, Y (BASELINE cfg4)."""
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(m, r, replace=False))
    cols = np.sort(rng.choice(n, r, replace=False))
    x = rng.integers(0, p, (m, r), dtype=np.int64)
    y = rng.integers(0, p, (r, n), dtype=np.int64)
    for k in range(r):
        x[: rows[k], k] = 0
        x[rows[k], k] = 1
        y[k, : cols[k]] = 0
        y[k, cols[k]] = 1
    return np.ascontiguousarray(_mulmod_exact(x, y, p)), rows, cols


def gen_cfg5(seed=0, n=65536, r=32768, p=65521):
    return gen_xy_rank(n, n, r, p, seed)


def effective_work(m, n, r) -> float:
    """BASELINE metric numerator W = 2mnr - (m+n) r^2 + 2 r^3 / 3."""
    return 2.0 * m * n * r - (m + n) * float(r) ** 2 + 2.0 * float(r) ** 3 / 3.0


def _pluq_batch_worker(args):
    """One process of pluq_batch: factor blocks[i] in place, return the per-block results."""
    blocks, p, threshold = args
    out = []
    for a in blocks:
        x = np.asarray(a).astype(field_dtype(p))
        c = Counts()
        pp, qq, r, _ = pluq(x, p, threshold, c)
        out.append((np.asarray(pp), np.asarray(qq), r, x.astype(np.int64), c.as_tuple()))
    return out


def pluq_batch(batch: np.ndarray, p: int, threshold: int = 30, processes: int | None = None):
    """The reference's per-matrix loop over a batch (cfg2), spread over a spawn-started
    process pool (each process single-threaded; one decomposition is
    single-threaded, distinct ones are independent).  Returns a list of
    (P.sigma, Q.sigma, r, packed int64, counts) per block."""
    import multiprocessing as mp
    import os

    n = len(batch)
    procs = max(1, min(processes or os.cpu_count() or 1, n))
    if procs == 1:
        return _pluq_batch_worker((batch, p, threshold))
    parts = np.array_split(np.arange(n), procs)
    env_old = os.environ.get("OPENBLAS_NUM_THREADS")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"  # inherited by the spawned children
    try:
        with mp.get_context("spawn").Pool(procs) as pool:
            res = pool.map(_pluq_batch_worker, [(batch[ix], p, threshold) for ix in parts])
    finally:
        if env_old is None:
            os.environ.pop("OPENBLAS_NUM_THREADS", None)
        else:
            os.environ["OPENBLAS_NUM_THREADS"] = env_old
    return [r for part in res for r in part]
