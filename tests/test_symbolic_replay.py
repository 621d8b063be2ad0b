"""Host symbolic replay of Algorithm 1 on a rank profile matrix (C ABI
pluq_rank_profile_replay, no GPU) against the oracle run on actual matrices.

The large-node pivot repair of the speculative LU (csrc/pluq_driver.cu speculative_lu)
takes P, Q and OpCounts from this replay; the facts it rests on (pluq_rpm.cuh): pluq(A)
and pluq(R_A) have the same P, Q, rank and OpCounts."""

import numpy as np
import pytest

from oracle import pluq_oracle as orc


@pytest.fixture(scope="module")
def lib():
    from paper_1301_4438_b200 import _native

    return _native.load_library(), _native


def _replay(lib, m, n, thr, pairs):
    lb, nat = lib
    r = len(pairs)
    pr = np.array([a for a, _ in pairs], np.int64)
    pc = np.array([b for _, b in pairs], np.int64)
    P = np.zeros(m, np.int64)
    Q = np.zeros(n, np.int64)
    cnt = np.zeros(4, np.int64)
    st = lb.pluq_rank_profile_replay(m, n, thr, r, nat.i64p(pr), nat.i64p(pc), nat.i64p(P), nat.i64p(Q), nat.i64p(cnt))
    return st, P, Q, tuple(int(v) for v in cnt)


def _rank_profile_matrix(a, p):
    """Support pairs of the oracle's pluq (= R_A)."""
    x = a.astype(orc.field_dtype(p))
    P, Q, r, c = orc.pluq(x, p, 30, orc.Counts())
    return orc.support_pairs(P, Q, r)


def _random_case(rng, p):
    m, n = int(rng.integers(1, 90)), int(rng.integers(1, 90))
    kind = rng.integers(0, 4)
    if kind == 0:
        a = rng.integers(0, p, (m, n))
    elif kind == 1:
        r = int(rng.integers(0, min(m, n) + 1))
        a = orc.gen_xy_rank(m, n, r, p, int(rng.integers(1 << 30)))
    elif kind == 2:
        r = int(rng.integers(1, min(m, n) + 1))
        if m < 2 or n < 2 or r > min(m, n):
            a = rng.integers(0, p, (m, n))
        else:
            a, _, _ = orc.gen_cfg4(seed=int(rng.integers(1 << 30)), m=m, n=n, r=r, p=p)
    else:  # sparse
        a = rng.integers(0, p, (m, n)) * (rng.random((m, n)) < 0.1)
    return np.asarray(a, np.int64)


@pytest.mark.parametrize("seed", range(6))
def test_replay_matches_oracle_on_random_matrices(lib, seed):
    rng = np.random.default_rng(seed)
    for _ in range(25):
        p = int(rng.choice([2, 3, 101, 65521]))
        a = _random_case(rng, p)
        m, n = a.shape
        for thr in (1, 3, 8, 30):
            x = a.astype(orc.field_dtype(p))
            c = orc.Counts()
            P, Q, r, _ = orc.pluq(x, p, thr, c)
            pairs = orc.support_pairs(P, Q, r)
            st, Ph, Qh, ch = _replay(lib, m, n, thr, pairs)
            assert st == 0
            assert np.array_equal(Ph, P) and np.array_equal(Qh, Q), (m, n, thr, p)
            assert ch == c.as_tuple(), (m, n, thr, p)


def test_replay_single_swap_like_cfg5(lib):
    """The structure the seed-0 cfg5 input has (one 2x2 column swap on an identity profile)
    at a size where the oracle can run the matrix itself."""
    p, n, g = 65521, 160, 57
    rng = np.random.default_rng(3)
    a = rng.integers(0, p, (n, n))
    # make leading minor g+1 vanish: row g restricted to columns :g+1 = a combination of the
    # rows above, the rest of row g random
    coef = rng.integers(0, p, g)
    a[g, :g + 1] = (coef @ a[:g, :g + 1].astype(object)) % p
    pairs = _rank_profile_matrix(a, p)
    assert (g, g + 1) in pairs and (g + 1, g) in pairs
    x = a.astype(np.float64)
    c = orc.Counts()
    P, Q, r, _ = orc.pluq(x, p, 30, c)
    st, Ph, Qh, ch = _replay(lib, n, n, 30, pairs)
    assert st == 0 and np.array_equal(Ph, P) and np.array_equal(Qh, Q) and ch == c.as_tuple()


def test_replay_rejects_non_permutation(lib):
    st, _, _, _ = _replay(lib, 4, 4, 30, [(0, 1), (1, 1)])
    assert st == 1
