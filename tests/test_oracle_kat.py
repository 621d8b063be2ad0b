"""Known-answer tests of the reference suite, restated against the oracle, plus
property checks (reconstruction, greedy rank profiles) — CPU only."""

import itertools

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import pluq_oracle as orc


def _greedy(rows, p):
    basis, kept = [], []
    for idx in range(rows.shape[0]):
        cur = rows[idx].astype(np.int64) % p
        for lead, vec in basis:
            c = cur[lead]
            if c:
                cur = (cur - c * vec) % p
        nz = np.flatnonzero(cur)
        if nz.size:
            lead = int(nz[0])
            basis.append((lead, (cur * pow(int(cur[lead]), -1, p)) % p))
            kept.append(idx)
    return tuple(kept)


def test_base_row_kat():  # test_recursive.py:65-74
    a = np.array([[0, 0, 5]], dtype=np.float64)
    P, Q, r, _ = orc.pluq(a, 7)
    assert r == 1 and a.tolist() == [[5, 0, 0]] and Q.tolist() == [2, 0, 1]


def test_base_col_kat():  # test_recursive.py:77-87
    a = np.array([[0], [2], [4]], dtype=np.float64)
    c = orc.Counts()
    P, Q, r, c = orc.pluq(a, 5, counts=c)
    assert r == 1 and a.ravel().tolist() == [2, 0, 2] and P.tolist() == [1, 0, 2]
    assert c.field_inv == 1 and c.field_mul == 1


def test_identity_kat():  # test_recursive.py:33-39
    a = np.eye(6)
    P, Q, r, _ = orc.pluq(a, 7, threshold=1)
    assert r == 6 and np.array_equal(P, np.arange(6)) and np.array_equal(a, np.eye(6))


def test_profiles_kat():  # test_recursive.py:42-47, README.md:132-141
    a = np.array([[0, 0], [1, 0]], dtype=np.float64)
    P, Q, r, _ = orc.pluq(a, 2, threshold=1)
    assert orc.leading_rank_profiles(P, Q, r, 2, 2) == ((1,), (0,))
    a = np.array([[0, 0, 3], [0, 2, 1], [0, 0, 5]], dtype=np.float64)
    P, Q, r, _ = orc.pluq(a, 1009)
    assert r == 2 and orc.leading_rank_profiles(P, Q, r, 2, 3) == ((0, 1), (1, 2))


def test_s_t_marker():  # test_recursive.py:125-141
    s = orc.s_perm(1, 1, 1, 1, 4, 8)
    tags = np.array([10, 10, 20, 20, 30, 30, 40, 40])
    assert tags[orc.perm_inverse(s)].tolist() == [10, 10, 30, 30, 20, 20, 40, 40]
    t = orc.t_perm(1, 1, 1, 1, 4, 9)
    tags = np.array([1, 3, 5, 5, 2, 4, 6, 6, 6])
    assert tags[t].tolist() == [1, 2, 3, 4, 5, 5, 6, 6, 6]


def test_exhaustive_3x3_f2():  # test_iterative.py:75-84
    for entries in itertools.product(range(2), repeat=9):
        a = np.array(entries, dtype=np.float64).reshape(3, 3)
        orig = a.astype(np.int64)
        P, Q, r, _ = orc.pluq_iterative(a, 2)
        assert np.array_equal(orc.reconstruct(a, P, Q, r, 2), orig)
        for k in range(4):
            for t in range(4):
                sub = orig[:k, :t]
                want = (_greedy(sub, 2), _greedy(sub.T, 2))
                assert orc.leading_rank_profiles(P, Q, r, k, t) == want


@settings(max_examples=60, deadline=None)
@given(p=st.sampled_from([2, 3, 101]), m=st.integers(0, 9), n=st.integers(0, 9),
       threshold=st.sampled_from([1, 2, 3, 30]), seed=st.integers(0, 2**32 - 1))
def test_reconstruction_and_profiles(p, m, n, threshold, seed):  # test_recursive.py:147-165
    a0 = np.random.default_rng(seed).integers(0, p, (m, n))
    a = a0.astype(np.float64)
    P, Q, r, _ = orc.pluq(a, p, threshold)
    assert np.array_equal(orc.reconstruct(a, P, Q, r, p), a0)
    assert r == len(_greedy(a0, p))
    for k in range(m + 1):
        for t in range(n + 1):
            sub = a0[:k, :t]
            assert orc.leading_rank_profiles(P, Q, r, k, t) == (_greedy(sub, p), _greedy(sub.T, p))


def test_threshold_must_be_positive():
    with pytest.raises(ValueError):
        orc.pluq(np.ones((1, 1)), 5, threshold=0)


def test_cfg4_generator_profiles():
    # the prescribed (I, J) are the row / column rank profiles by construction
    a, rows, cols = orc.gen_cfg4(seed=1, m=96, n=160, r=40, p=8388593)
    P, Q, r, _ = orc.pluq(a.copy(), 8388593)
    assert r == 40
    assert orc.row_rank_profile(P, Q, r) == tuple(int(v) for v in rows)
    assert orc.col_rank_profile(P, Q, r) == tuple(int(v) for v in cols)


def test_effective_work_matches_counted_work_on_generic_input():
    # W matches the counted mul+add within ~0.2% on generic-profile input
    a = orc.gen_cfg1(seed=0, m=128, n=128, r=96)
    c = orc.Counts()
    orc.pluq(a.astype(np.float64), 65521, counts=c)
    w = orc.effective_work(128, 128, 96)
    assert abs((c.field_mul + c.field_add) - w) / w < 0.03
