"""The device generators draw the SURVEY §8(d) PCG64 stream (CPU checks of the host side).

paper_1301_4438_b200/gen.py draws each uniform matrix as int32 row chunks; these tests pin
that this is the same stream as the oracle's single int64 draw (oracle/pluq_oracle.py
gen_*), for both BASELINE primes, odd chunk sizes (the 32-bit half-draw buffer carries over
between calls) and the draws that follow (permutations, rng.choice).
"""

import numpy as np
import pytest

from oracle import pluq_oracle as orc
from paper_1301_4438_b200.gen import row_chunks


@pytest.mark.parametrize("p", [65521, 8388593, 2, 101])
@pytest.mark.parametrize("chunk", [1, 7, 333, 1 << 20])
def test_chunked_int32_draws_equal_int64_stream(p, chunk):
    rows, cols = 37, 29
    a = np.random.default_rng(5).integers(0, p, (rows, cols), dtype=np.int64)
    b = np.random.default_rng(5).integers(0, p, (cols, rows), dtype=np.int64)
    rng = np.random.default_rng(5)
    got_a = np.concatenate([blk for _, blk in row_chunks(rng, rows, cols, p, chunk)])
    got_b = np.concatenate([blk for _, blk in row_chunks(rng, cols, rows, p, chunk)])
    assert got_a.dtype == np.int32
    assert np.array_equal(got_a, a)
    ref = np.random.default_rng(5)
    ref.integers(0, p, (rows, cols), dtype=np.int64)
    assert np.array_equal(got_b, ref.integers(0, p, (cols, rows), dtype=np.int64))
    # the generator state after the chunked draws equals the state after the single draws
    ref2 = np.random.default_rng(5)
    ref2.integers(0, p, (rows, cols), dtype=np.int64)
    ref2.integers(0, p, (cols, rows), dtype=np.int64)
    assert np.array_equal(rng.permutation(50), ref2.permutation(50))


def _host_xy_rank(m, n, r, p, seed, chunk):
    """gen_xy_rank_device's draw order with the product and gathers done by the oracle."""
    rng = np.random.default_rng(seed)
    x = np.concatenate([blk for _, blk in row_chunks(rng, m, r, p, chunk)]).astype(np.int64)
    y = np.concatenate([blk for _, blk in row_chunks(rng, r, n, p, chunk)]).astype(np.int64)
    a = orc._mulmod_exact(x, y, p)
    return a[rng.permutation(m)][:, rng.permutation(n)]


def test_xy_rank_order_matches_oracle():
    for m, n, r, p, seed in ((64, 48, 20, 65521, 0), (40, 72, 33, 8388593, 3)):
        assert np.array_equal(_host_xy_rank(m, n, r, p, seed, 101), orc.gen_xy_rank(m, n, r, p, seed))


def test_cfg4_order_matches_oracle():
    m, n, r, p, seed = 48, 96, 16, 8388593, 2
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(m, r, replace=False))
    cols = np.sort(rng.choice(n, r, replace=False))
    x = np.concatenate([blk for _, blk in row_chunks(rng, m, r, p, 77)]).astype(np.int64)
    y = np.concatenate([blk for _, blk in row_chunks(rng, r, n, p, 77)]).astype(np.int64)
    x[np.arange(m)[:, None] < rows[None, :]] = 0
    x[rows, np.arange(r)] = 1
    y[np.arange(n)[None, :] < cols[:, None]] = 0
    y[np.arange(r), cols] = 1
    a0, rows0, cols0 = orc.gen_cfg4(seed=seed, m=m, n=n, r=r, p=p)
    assert np.array_equal(rows, rows0) and np.array_equal(cols, cols0)
    assert np.array_equal(orc._mulmod_exact(x, y, p), a0)


def test_cfg2_cfg3_order_matches_oracle():
    b = np.concatenate([blk for _, blk in row_chunks(np.random.default_rng(4), 6 * 16, 16, 65521, 50)])
    assert np.array_equal(b.reshape(6, 16, 16), orc.gen_cfg2(seed=4, batch=6, m=16, n=16))
    c = np.concatenate([blk for _, blk in row_chunks(np.random.default_rng(9), 40, 40, 65521, 123)])
    assert np.array_equal(c, orc.gen_cfg3(seed=9, n=40))
