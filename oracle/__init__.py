"""TEST INFRASTRUCTURE ONLY — CPU oracle for the PLUQ-mod-p hot path.

This package is a numpy restatement of the reference algorithm
(`/root/reference/pkg/src/pluq/recursive.py`, `iterative.py`, `kernels.py`,
`field.py`, `matrix.py`).  It exists to CHECK the CUDA product path and to be
timed as the CPU baseline in `bench.py --impl reference`.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu-baseline leg may
import it.  The product package `paper_1301_4438_b200` never imports it.

Parity pinning: `tests/golden/make_golden.py` runs the real reference package
(importable in the build container from `/root/reference/pkg/src`) and stores
its outputs as fixtures; `tests/test_oracle_golden.py` checks this oracle
against every one of them (P, Q, r, packed, OpCounts), plus the reference's own
known-answer tests restated in `tests/test_oracle_kat.py`.
"""

from .pluq_oracle import *  # noqa: F401,F403
