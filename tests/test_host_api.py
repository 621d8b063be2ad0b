"""Host-side logic of the drop-in API and the C-ABI library (no GPU compute)."""

import os
import re

import numpy as np
import pytest

import paper_1301_4438_b200 as pb
from paper_1301_4438_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.load_library()
    header = open(os.path.join(ROOT, "include", "pluq_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(pluq_\w+)\s*\(", header, re.M))
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, name


def test_public_api_mirrors_reference_names():
    # the factorization-path surface of pluq/__init__.py:9-88
    for name in ["pluq", "pluq_iterative", "PluqFactors", "Permutation", "DenseMatrix", "OpCounts",
                 "PrimeField", "row_rank_profile", "col_rank_profile", "leading_rank_profiles",
                 "apply_rows", "apply_cols", "perm_block_diag", "build_s_perm", "build_t_perm",
                 "base_case_row", "base_case_col", "Workspace", "TrackingWorkspace", "DEFAULT_THRESHOLD",
                 "inverse_mod", "is_prime"]:
        assert hasattr(pb, name), name
    assert pb.DEFAULT_THRESHOLD == 30


def test_field_validation_and_dtype():  # field.py:65-81
    with pytest.raises(ValueError):
        pb.PrimeField(91)
    with pytest.raises(ValueError):
        pb.PrimeField(67108879)  # prime above 2^26 without the override
    assert pb.PrimeField(67108879, allow_large_modulus=True).dtype == np.int64
    assert pb.PrimeField(65521).dtype == np.float64
    assert pb.PrimeField(8388593).dtype == np.int64
    assert pb.PrimeField(65521).limbs == 2 and pb.PrimeField(8388593).limbs == 3 and pb.PrimeField(251).limbs == 1
    with pytest.raises(ValueError):
        pb.DenseMatrix(pb.PrimeField(5), np.array([[5]]))
    with pytest.raises(ZeroDivisionError):
        pb.inverse_mod(0, 7)
    assert pb.inverse_mod(3, 7) == 5


def test_threshold_validation_before_any_device_work():
    with pytest.raises(ValueError):
        pb.pluq(pb.DenseMatrix(pb.PrimeField(5), np.array([[1]])), threshold=0)


def test_block_permutations():  # test_recursive.py:107-141
    assert pb.build_s_perm(0, 0, 0, 0, 3, 7).is_identity()
    assert pb.build_t_perm(0, 0, 0, 0, 3, 7).is_identity()
    assert pb.build_s_perm(4, 0, 0, 4, 4, 8).is_identity()
    assert pb.build_t_perm(4, 0, 0, 4, 4, 8).is_identity()
    with pytest.raises(ValueError):
        pb.build_s_perm(3, 2, 0, 0, 4, 8)
    with pytest.raises(ValueError):
        pb.build_t_perm(0, 3, 0, 2, 4, 8)
    s = pb.build_s_perm(1, 1, 1, 1, 4, 8)
    tags = np.array([10, 10, 20, 20, 30, 30, 40, 40])
    assert tags[s.inverse().sigma].tolist() == [10, 10, 30, 30, 20, 20, 40, 40]
    t = pb.build_t_perm(1, 1, 1, 1, 4, 9)
    tags = np.array([1, 3, 5, 5, 2, 4, 6, 6, 6])
    assert tags[t.sigma].tolist() == [1, 2, 3, 4, 5, 5, 6, 6, 6]


def test_block_permutations_match_oracle_exhaustively():
    from oracle import pluq_oracle as orc

    for m in range(0, 7):
        for k in range(0, m + 1):
            for r1 in range(0, k + 1):
                for r2 in range(0, k - r1 + 1):
                    for r3 in range(0, m - k + 1):
                        for r4 in range(0, m - k - r3 + 1):
                            assert np.array_equal(pb.build_s_perm(r1, r2, r3, r4, k, m).sigma,
                                                  orc.s_perm(r1, r2, r3, r4, k, m))
                            if r1 + r3 <= k and r2 + r4 <= m - k:
                                assert np.array_equal(pb.build_t_perm(r1, r2, r3, r4, k, m).sigma,
                                                      orc.t_perm(r1, r2, r3, r4, k, m))


def test_permutation_algebra():  # matrix.py:161-246
    p = pb.Permutation([2, 0, 1])
    assert p.compose(p.inverse()).is_identity()
    assert p.inverse().sigma.tolist() == [1, 2, 0]
    with pytest.raises(ValueError):
        pb.Permutation([0, 0, 1])
    d = pb.perm_block_diag([pb.Permutation([1, 0]), pb.Permutation([0])])
    assert d.sigma.tolist() == [1, 0, 2]
    a = np.arange(9).reshape(3, 3).astype(np.float64)
    pb.apply_rows(a, p)
    assert a[:, 0].tolist() == [6, 0, 3]


def test_rank_profile_extraction_is_host_side():
    f = pb.PluqFactors(pb.Permutation([1, 0]), pb.Permutation([0, 1]), 1,
                       pb.DenseMatrix(pb.PrimeField(2), np.array([[1, 0], [0, 0]])))
    assert pb.row_rank_profile(f) == (1,)
    assert pb.col_rank_profile(f) == (0,)
    assert pb.leading_rank_profiles(f, 2, 2) == ((1,), (0,))
    assert pb.leading_rank_profiles(f, 1, 2) == ((), ())
    with pytest.raises(ValueError):
        pb.leading_rank_profiles(f, 3, 0)
