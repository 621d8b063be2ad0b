"""The generic-rank-profile fast path (CPU-checkable pieces).

Claim used by the speculative no-pivot path: if the leading principal minors of
orders 1..r are nonzero and the Schur complement after r pivots is zero, the
reference recursion returns P = Q = I, rank r and the unique unpivoted LU factors,
for every threshold; and its OpCounts depend only on (m, n, r, threshold)."""

import numpy as np

from oracle import pluq_oracle as orc
from paper_1301_4438_b200 import _native


def _unpivoted(a, p):
    a = a.astype(np.int64) % p
    m, n = a.shape
    for t in range(min(m, n)):
        piv = int(a[t, t])
        if piv == 0:
            return (not a[t:, t:].any()), t, a
        inv = pow(piv, -1, p)
        a[t + 1:, t] = a[t + 1:, t] * inv % p
        a[t + 1:, t + 1:] = (a[t + 1:, t + 1:] - np.outer(a[t + 1:, t], a[t, t + 1:])) % p
    return True, min(m, n), a


def test_generic_profile_claim_and_counts():
    lib = _native.load_library()
    rng = np.random.default_rng(7)
    generic = 0
    for trial in range(260):
        p = int(rng.choice([2, 3, 101, 65521]))
        m, n = (int(x) for x in rng.integers(1, 60, 2))
        r = int(rng.integers(0, min(m, n) + 1))
        a = rng.integers(0, p, (m, n)) if trial % 3 == 0 else orc.gen_xy_rank(m, n, r, p, trial, permute=trial % 3 == 2)
        thr = int(rng.choice([1, 2, 4, 30, 10**9]))  # 10**9: Algorithm 2 on the whole matrix
        ok, rr, packed = _unpivoted(a, p)
        if not ok:
            continue
        generic += 1
        x = a.astype(orc.field_dtype(p))
        c = orc.Counts()
        P, Q, R, c = orc.pluq(x, p, thr, c)
        assert R == rr
        assert np.array_equal(P, np.arange(m)) and np.array_equal(Q, np.arange(n))
        assert np.array_equal(x.astype(np.int64), packed)
        out = np.zeros(4, dtype=np.int64)
        assert lib.pluq_generic_counts(m, n, rr, thr, _native.i64p(out)) == 0
        assert tuple(int(v) for v in out) == c.as_tuple(), (m, n, rr, thr)
    assert generic > 80
