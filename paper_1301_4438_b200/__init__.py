"""B200-native rank-profile-revealing PLUQ over GF(p) (arXiv:1301.4438 hot path).

Drop-in for the reference package ``pluq`` (/root/reference/pkg/src/pluq/__init__.py:9-88)
on the factorization path: same entry points, types, in-place contract, OpCounts
charges and bit-exact (P, Q, packed, rank) results, computed by hand-written
sm_100a CUDA in ``libpluq_b200.so`` (C ABI: include/pluq_b200.h).
"""

from .field import ABSOLUTE_MODULUS_BOUND, DEFAULT_MODULUS_BOUND, PrimeField, inverse_mod, is_prime
from .kernels import ClassicalKernels, CudaKernels, device_matmul_mod
from .matrix import DenseMatrix, OpCounts, Permutation, PluqFactors, apply_cols, apply_rows, perm_block_diag
from .distributed import pluq_distributed
from .leu import LeuFactors, check_triangular_extension, to_leu
from .rank_profile import col_rank_profile, leading_rank_profiles, row_rank_profile
from .recursive import (
    DEFAULT_THRESHOLD,
    BatchedPluq,
    TrackingWorkspace,
    Workspace,
    base_case_col,
    base_case_row,
    build_s_perm,
    build_t_perm,
    last_stats,
    pluq,
    pluq_batched,
    pluq_iterative,
)

__version__ = "0.1.0"

__all__ = [
    "ABSOLUTE_MODULUS_BOUND",
    "BatchedPluq",
    "ClassicalKernels",
    "CudaKernels",
    "DEFAULT_MODULUS_BOUND",
    "DEFAULT_THRESHOLD",
    "DenseMatrix",
    "LeuFactors",
    "OpCounts",
    "Permutation",
    "PluqFactors",
    "PrimeField",
    "TrackingWorkspace",
    "Workspace",
    "apply_cols",
    "apply_rows",
    "base_case_col",
    "base_case_row",
    "build_s_perm",
    "build_t_perm",
    "check_triangular_extension",
    "col_rank_profile",
    "device_matmul_mod",
    "inverse_mod",
    "is_prime",
    "last_stats",
    "leading_rank_profiles",
    "perm_block_diag",
    "pluq",
    "pluq_batched",
    "pluq_distributed",
    "pluq_iterative",
    "row_rank_profile",
    "to_leu",
]
