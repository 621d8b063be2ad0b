"""Pivot repair of the speculative LU on large nodes (csrc/pluq_driver.cu speculative_lu).

A leading minor that vanishes by coincidence (probability ~ r/p per matrix: the seed-0
cfg5 input has one, at pivot 11148) used to send the whole node to the exact recursion.
Now the zero pivot is repaired by the row-order elimination that defines R_A (the
leftmost nonzero column of the pivot row is rotated into place) and Alg.1 is replayed
symbolically on R_A for P, Q and the OpCounts.  Every case is compared bit for bit with the
oracle (P, Q, rank, packed, OpCounts)."""

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


def _vanish(a, g, width, p, rng):
    """Make the leading minors g+1 .. g+width of a vanish in the first `width` columns of
    row g: row g restricted to columns :g+width = a combination of the rows above."""
    coef = rng.integers(0, p, g).astype(object)
    a[g, :g + width] = np.array((coef @ a[:g, :g + width].astype(object)) % p, dtype=np.int64)


CASES = [
    # name, m, n, rank or None, [(g, width)], p
    ("mid_block", 400, 420, None, [(57, 1)], 65521),
    ("block_edge", 400, 400, None, [(127, 1)], 65521),
    ("block_start", 400, 400, None, [(128, 1)], 65521),
    ("panel_edge", 600, 640, None, [(255, 1)], 65521),
    ("second_panel", 600, 600, None, [(300, 1)], 65521),
    ("two", 520, 500, None, [(40, 1), (333, 1)], 65521),
    ("wide_gap", 300, 360, None, [(90, 3)], 65521),
    ("near_end", 300, 300, None, [(297, 1)], 65521),
    ("rank_deficient", 420, 400, 250, [(100, 1)], 65521),
    ("p23", 360, 380, None, [(70, 1)], 8388593),
    ("small_p", 300, 300, None, [(20, 1)], 1009),
]


def _make(name, m, n, r, gs, p):
    rng = np.random.default_rng(m * 7 + n)
    a = rng.integers(0, p, (m, n)) if r is None else orc.gen_xy_rank(m, n, r, p, 5)
    a = np.asarray(a, np.int64)
    for g, w in gs:
        _vanish(a, g, w, p, rng)
    return a


@pytest.mark.parametrize("opts", [dict(small_cap=1, spec_panel=256),
                                  dict(small_cap=1, spec_block=16, spec_panel=48, spec_check=3)],
                         ids=["blocks128", "blocks16"])
@pytest.mark.parametrize("name,m,n,r,gs,p", CASES, ids=[c[0] for c in CASES])
def test_repair_vs_oracle(pb, opts, name, m, n, r, gs, p):
    from paper_1301_4438_b200 import _native

    a0 = _make(name, m, n, r, gs, p)
    x = a0.astype(orc.field_dtype(p))
    cc = orc.Counts()
    P, Q, R, _ = orc.pluq(x, p, 30, cc)
    ctx = _native.context()
    old = {k: ctx.get_option(k) for k in opts}
    for k, v in opts.items():
        ctx.set_option(k, v)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(orc.field_dtype(p)))
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        st = pb.last_stats()
    finally:
        for k, v in old.items():
            ctx.set_option(k, v)
    assert f.rank == R
    assert np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(a.data, x)
    assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == cc.as_tuple()
    # the top node was finished by the repaired speculative LU, not the exact recursion
    assert st["spec_repairs"] >= 1 and st["speculative_fail"] == 0, st


def test_repair_disabled_falls_back(pb):
    from paper_1301_4438_b200 import _native

    p = 65521
    a0 = _make("mid_block", 400, 420, None, [(57, 1)], p)
    x = a0.astype(np.float64)
    P, Q, R, _ = orc.pluq(x, p, 30, orc.Counts())
    ctx = _native.context()
    ctx.set_option("small_cap", 1)
    ctx.set_option("spec_repairs", 0)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(np.float64))
        f = pb.pluq(a)
        st = pb.last_stats()
    finally:
        ctx.set_option("small_cap", 128 * 128)
        ctx.set_option("spec_repairs", 32)
    assert st["speculative_fail"] >= 1 and st["spec_repairs"] == 0
    assert f.rank == R and np.array_equal(f.q_perm.sigma, Q) and np.array_equal(a.data, x)


def test_cfg5_seed0_full_size_repaired(pb):
    """The headline input itself (65536^2, rank 32768, seed 0): one coincidence at pivot
    11148, repaired; Q swaps columns 11148/11149 (the reference's rank profile), P = I."""
    import torch
    from paper_1301_4438_b200 import gen, verify

    a5 = gen.gen_cfg5_device(seed=0)
    f = pb.pluq(pb.DenseMatrix(pb.PrimeField(65521), a5.clone()))
    st = pb.last_stats()
    assert f.rank == 32768 and st["spec_repairs"] == 1 and st["speculative_fail"] == 0
    q = np.arange(65536)
    q[11148], q[11149] = 11149, 11148
    assert np.array_equal(f.p_perm.sigma, np.arange(65536)) and np.array_equal(f.q_perm.sigma, q)
    assert verify.structure_ok(f) and verify.freivalds(a5, f, probes=2)
    del a5, f
    torch.cuda.empty_cache()


PAIR_CASES = [
    # name, m, n, rank or None, [(g, width)]: zero pivots in the first / second panel of a pair
    ("generic", 1100, 1200, None, []),
    ("stop_second_of_pair", 1100, 1100, 400, []),      # rank 400: zero Schur inside panel 1 (W=256)
    ("stop_first_of_pair", 1100, 1100, 600, []),       # inside panel 2
    ("repair_second_of_pair", 1100, 1150, None, [(300, 1)]),
    ("repair_two_pairs", 1200, 1100, None, [(100, 1), (700, 1)]),
]


@pytest.mark.parametrize("inner_la,panel_rec", [(0, 0), (1, 0), (0, 2)], ids=["rl", "rl_la", "rec"])
@pytest.mark.parametrize("la_pair", [0, 1, 2, 3])
@pytest.mark.parametrize("name,m,n,r,gs", PAIR_CASES, ids=[c[0] for c in PAIR_CASES])
def test_paired_far_updates_vs_oracle(pb, la_pair, name, m, n, r, gs, inner_la, panel_rec):
    """Panel P's far update merged into panel P+1's (option la_pair, one K = 2W GEMM), with
    zero pivots / repairs in either panel of a pair (the finishing step applies a pending
    deferred update)."""
    from paper_1301_4438_b200 import _native

    p = 65521
    a0 = _make(name, m, n, r, gs, p)
    x = a0.astype(np.float64)
    cc = orc.Counts()
    P, Q, R, _ = orc.pluq(x, p, 30, cc)
    ctx = _native.context()
    opts = dict(small_cap=1, spec_panel=256, la_pair=la_pair, inner_la=inner_la, panel_rec=panel_rec)
    old = {k: ctx.get_option(k) for k in opts}
    for k, v in opts.items():
        ctx.set_option(k, v)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(np.float64))
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        st = pb.last_stats()
    finally:
        for k, v in old.items():
            ctx.set_option(k, v)
    assert st["speculative_ok"] >= 1 and st["speculative_fail"] == 0
    assert f.rank == R and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(a.data, x)
    assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == cc.as_tuple()


@pytest.mark.parametrize("panel_rec", [0, 2])
@pytest.mark.parametrize("la_pair", [0, 1, 2, 3])
@pytest.mark.parametrize("W", [384, 640, 768])
def test_panel_widths_generic_and_repaired(pb, la_pair, W, panel_rec):
    """Panel widths that do not divide the size (partial last panels, pairs cut short), on a
    rank-deficient X Y input with one coincidental zero minor: the speculative path must
    succeed (no fallback) and match the oracle."""
    from paper_1301_4438_b200 import _native

    p, m, n = 65521, 2000, 2100
    a0 = _make("w", m, n, 1300, [(500, 1)], p)
    x = a0.astype(np.float64)
    cc = orc.Counts()
    P, Q, R, _ = orc.pluq(x, p, 30, cc)
    ctx = _native.context()
    opts = dict(small_cap=1, spec_panel=W, la_pair=la_pair, panel_rec=panel_rec)
    old = {k: ctx.get_option(k) for k in opts}
    for k, v in opts.items():
        ctx.set_option(k, v)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(np.float64))
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        st = pb.last_stats()
    finally:
        for k, v in old.items():
            ctx.set_option(k, v)
    assert f.rank == R and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(a.data, x)
    assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == cc.as_tuple()
    assert st["speculative_fail"] == 0 and st["spec_repairs"] == 1, st


@pytest.mark.parametrize("par_trsm", [0, 1])
@pytest.mark.parametrize("r,gs", [(130, []), (300, []), (520, []), (777, []), (1000, []), (1024, []), (None, [(5, 1)]),
                                  (None, [(200, 1), (640, 2)]), (None, [(895, 1)]), (None, [(1023, 1)]),
                                  (1100, [(384, 1)])])
def test_recursive_panel_stops(pb, r, gs, par_trsm):
    """Recursive panel factorization (option panel_rec) on 1024-wide panels (3 levels of
    halving): zero pivots / zero Schur complements at every depth of the recursion — the
    finishing step applies the updates of the nodes skipped under the stop flag."""
    from paper_1301_4438_b200 import _native

    p, m, n = 65521, 1400, 1300
    a0 = _make("rp", m, n, r, gs, p)
    x = a0.astype(np.float64)
    cc = orc.Counts()
    P, Q, R, _ = orc.pluq(x, p, 30, cc)
    ctx = _native.context()
    opts = dict(small_cap=1, spec_panel=1024, panel_rec=2, par_trsm=par_trsm, spec_check=3)
    old = {k: ctx.get_option(k) for k in opts}
    for k, v in opts.items():
        ctx.set_option(k, v)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(np.float64))
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        st = pb.last_stats()
    finally:
        for k, v in old.items():
            ctx.set_option(k, v)
    assert st["speculative_ok"] >= 1 and st["speculative_fail"] == 0, st
    assert f.rank == R and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(a.data, x)
    assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == cc.as_tuple()


@pytest.mark.parametrize("first_single", [0, 1])
@pytest.mark.parametrize("preinv", [0, 1])
@pytest.mark.parametrize("name,m,n,r,gs", PAIR_CASES + [("repair_first_panel", 1300, 1300, None, [(77, 1)]),
                                                         ("rank_in_third", 1300, 1250, 700, [])],
                         ids=[c[0] for c in PAIR_CASES] + ["repair_first_panel", "rank_in_third"])
def test_group_lookahead_variants(pb, name, m, n, r, gs, first_single, preinv):
    """Group look-ahead (la_pair = 2) with the first panel grouped or alone (la_first_single) and
    with / without the panel inverses formed ahead (la_preinv; 256-wide panels take the
    precomputed-inverse GEMM form), far update split in two parts."""
    from paper_1301_4438_b200 import _native

    p = 65521
    a0 = _make(name, m, n, r, gs, p)
    x = a0.astype(np.float64)
    cc = orc.Counts()
    P, Q, R, _ = orc.pluq(x, p, 30, cc)
    ctx = _native.context()
    opts = dict(small_cap=1, spec_panel=256, la_pair=2, panel_rec=2, la_first_single=first_single, la_preinv=preinv)
    old = {k: ctx.get_option(k) for k in opts}
    for k, v in opts.items():
        ctx.set_option(k, v)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(np.float64))
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        st = pb.last_stats()
    finally:
        for k, v in old.items():
            ctx.set_option(k, v)
    assert st["speculative_ok"] >= 1 and st["speculative_fail"] == 0
    assert f.rank == R and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(a.data, x)
    assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == cc.as_tuple()


UNFACTOR_CASES = [
    # name, m, n, zero rows (rows without a pivot: the speculation must fail there), coincidences, p, repairs allowed
    ("zero_row_early", 500, 520, [3], [], 65521, 32),
    ("zero_row_late", 500, 500, [300], [], 65521, 32),
    ("zero_row_block_edge", 640, 600, [255], [], 65521, 32),
    ("repair_then_zero_row", 600, 640, [350], [(100, 1)], 65521, 32),
    ("two_repairs_then_zero_row", 700, 700, [520], [(60, 1), (300, 2)], 65521, 32),
    ("coincidence_no_repairs", 400, 420, [], [(57, 1)], 65521, 0),
    ("p23_zero_row", 380, 400, [200], [], 8388593, 32),
    ("tall_zero_row", 900, 300, [150], [], 65521, 32),
    ("wide_zero_row", 300, 900, [150], [], 65521, 32),
]


@pytest.mark.parametrize("name,m,n,zrows,gs,p,reps", UNFACTOR_CASES, ids=[c[0] for c in UNFACTOR_CASES])
def test_unfactor_restores_without_backup(pb, name, m, n, zrows, gs, p, reps):
    """spec_backup = 0: a failed speculative LU re-multiplies its partial factors in place
    (Ops::unfactor: A22 = S + L21 U12, A12 = L11 U12, A21 = L21 U11, A11 = L11 U11) and undoes
    the repairs' column rotations instead of copying a backup back; the exact recursion that
    follows must then see the original matrix — bit-exact against the oracle."""
    from paper_1301_4438_b200 import _native

    rng = np.random.default_rng(m * 13 + n)
    a0 = np.asarray(rng.integers(0, p, (m, n)), np.int64)
    for g, w in gs:
        _vanish(a0, g, w, p, rng)
    for zr in zrows:  # row zr = combination of the rows above: no pivot in that row
        coef = rng.integers(0, p, zr).astype(object)
        a0[zr, :] = np.array((coef @ a0[:zr, :].astype(object)) % p, dtype=np.int64) if zr else 0
    x = a0.astype(orc.field_dtype(p))
    cc = orc.Counts()
    P, Q, R, _ = orc.pluq(x, p, 30, cc)
    ctx = _native.context()
    opts = dict(small_cap=1, spec_panel=256, spec_repairs=reps, spec_backup=0)
    old = {k: ctx.get_option(k) for k in opts}
    for k, v in opts.items():
        ctx.set_option(k, v)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(orc.field_dtype(p)))
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        st = pb.last_stats()
    finally:
        for k, v in old.items():
            ctx.set_option(k, v)
    assert st["speculative_fail"] >= 1, st
    assert f.rank == R and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(a.data, x)
    assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == cc.as_tuple()
