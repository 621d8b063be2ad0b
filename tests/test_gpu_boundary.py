"""Error behaviour and hygiene at the C-ABI boundary (SURVEY §8(b) error conventions).

The reference rejects non-canonical entries when a DenseMatrix is built
(/root/reference/pkg/src/pluq/field.py:140-147, ValueError) before anything is modified;
the device paths do the same through the range check in the C ABI.
"""

import ctypes
import time

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


@pytest.mark.parametrize("bad", [65521, 70000, -1, -65521])
def test_device_densematrix_rejects_noncanonical(pb, bad):
    import torch

    t = torch.randint(0, 65521, (300, 200), dtype=torch.int32, device="cuda")
    t[123, 77] = bad
    with pytest.raises(ValueError):
        pb.DenseMatrix(pb.PrimeField(65521), t)


@pytest.mark.parametrize("m,n,p,where", [(256, 256, 65521, (200, 3)), (1000, 1200, 65521, (999, 1199)),
                                         (700, 500, 8388593, (0, 0)), (100, 40, 65521, (50, 39))])
def test_c_abi_factor_rejects_and_leaves_input(pb, m, n, p, where):
    """Non-canonical entries: PLUQ_EINVAL with the input untouched, whether the check runs
    before the factorization or inside the top node's backup copy (large nodes)."""
    import torch
    from paper_1301_4438_b200 import _native

    t = torch.randint(0, p, (m, n), dtype=torch.int32, device="cuda")
    t[where] = p + 5
    before = t.clone()
    ctx = _native.context()
    psig = np.zeros(m, np.int64)
    qsig = np.zeros(n, np.int64)
    rank = np.zeros(1, np.int64)
    st = ctx.lib.pluq_factor(ctx.handle, t.data_ptr(), n, m, n, p, 30, _native.i64p(psig),
                             _native.i64p(qsig), _native.i64p(rank), None)
    assert st == _native.PLUQ_EINVAL
    assert torch.equal(t, before)
    t[where] = 1  # and the same matrix with a valid entry factors fine
    st = ctx.lib.pluq_factor(ctx.handle, t.data_ptr(), n, m, n, p, 30, _native.i64p(psig),
                             _native.i64p(qsig), _native.i64p(rank), None)
    assert st == _native.PLUQ_OK


@pytest.mark.parametrize("dtype,bad", [(np.float64, 0.5), (np.float64, float("nan")), (np.float64, -3.0),
                                       (np.float64, 65521.0), (np.int64, 65521), (np.int64, -2)])
def test_c_abi_host_buffers_reject_and_leave_input(pb, dtype, bad):
    from paper_1301_4438_b200 import _native

    p = 65521
    a = np.random.default_rng(1).integers(0, p, (150, 170)).astype(dtype)
    a[17, 33] = bad
    before = a.copy()
    ctx = _native.context()
    psig = np.zeros(150, np.int64)
    qsig = np.zeros(170, np.int64)
    rank = np.zeros(1, np.int64)
    fn = ctx.lib.pluq_factor_host_f64 if dtype == np.float64 else ctx.lib.pluq_factor_host_i64
    st = fn(ctx.handle, a.ctypes.data, 150, 170, p, 30, _native.i64p(psig), _native.i64p(qsig), _native.i64p(rank), None)
    assert st == _native.PLUQ_EINVAL
    assert np.array_equal(a, before, equal_nan=True)


def test_batched_rejects_noncanonical(pb):
    import torch

    t = torch.randint(0, 65521, (64, 64, 64), dtype=torch.int32, device="cuda")
    t[40, 5, 6] = -7
    before = t.clone()
    with pytest.raises(ValueError):
        pb.pluq_batched(t, 65521, 30)
    assert torch.equal(t, before)
    h = np.random.default_rng(2).integers(0, 65521, (32, 64, 64)).astype(np.float64)
    h[31, 63, 63] = 1e9
    with pytest.raises(ValueError):
        pb.pluq_batched(h, 65521, 30)
    # streaming-size batch (concurrent fallback consumers): the asynchronous check aborts every
    # kernel of the call, the input stays untouched, and the next call is unaffected
    big = torch.randint(0, 65521, (2048, 64, 64), dtype=torch.int32, device="cuda")
    good = big.clone()
    big[2047, 63, 0] = 65521
    before = big.clone()
    t0 = time.perf_counter()
    with pytest.raises(ValueError):
        pb.pluq_batched(big, 65521, 30)
    torch.cuda.synchronize()
    assert time.perf_counter() - t0 < 1.0
    assert torch.equal(big, before)
    res = pb.pluq_batched(good, 65521, 30)
    torch.cuda.synchronize()
    assert int(res.ranks.min()) >= 60


def test_current_device_and_options_roundtrip(pb):
    import torch
    from paper_1301_4438_b200 import _native

    torch.cuda.set_device(0)
    a = pb.DenseMatrix(pb.PrimeField(101), torch.randint(0, 101, (64, 80), dtype=torch.int32, device="cuda"))
    pb.pluq(a)
    assert torch.cuda.current_device() == 0
    ctx = _native.context()
    old = ctx.get_option("spec_panel")
    ctx.set_option("spec_panel", 512)
    assert ctx.get_option("spec_panel") == 512
    ctx.set_option("spec_panel", old)
    with pytest.raises(ValueError):
        ctx.get_option("no_such_option")


def test_classical_kernels_alias(pb):
    assert pb.ClassicalKernels is pb.CudaKernels
    k = pb.ClassicalKernels(pb.PrimeField(65521))
    assert hasattr(k, "mm_acc") and hasattr(k, "trsm_left_unit_lower") and hasattr(k, "trsm_right_upper")


@pytest.mark.parametrize("m,n", [(48, 48), (40, 56)])
def test_streaming_batch_non_64_blocks_bounded_time(pb, m, n):
    """Batches of >= 1024 blocks run the concurrent rank-profile consumer; for shapes other
    than 64x64 (crout_fast_kernel) it must see every generic CTA finish and exit at once
    instead of waiting out its spin bound."""
    import torch

    p = 65521
    host = np.random.default_rng(m * n).integers(0, p, (1536, m, n))
    host[::97] = np.stack([orc.gen_xy_rank(m, n, 10, p, s) for s in range(0, 1536, 97)])  # non-generic blocks
    t = torch.from_numpy(host).cuda().to(torch.int32)
    w = t.clone()
    pb.pluq_batched(w, p, 30)  # warm-up (module load, attributes)
    torch.cuda.synchronize()
    w.copy_(t)
    t0 = time.perf_counter()
    res = pb.pluq_batched(w, p, 30)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    assert dt < 0.05, dt
    for b in list(range(0, 1536, 97)) + [1, 500, 1535]:
        P, Q, r, _ = orc.pluq(host[b].astype(np.float64), p, 30)
        assert int(res.ranks[b]) == r and np.array_equal(res.p_sigma[b].cpu().numpy(), P)


@pytest.mark.parametrize("p,dtype", [(65521, np.float64), (8388593, np.int64)])
def test_host_pipeline_chunks_vs_oracle(pb, p, dtype):
    """Large host matrices go through the pinned-ring pipeline (host threads convert to
    uint32 while DMA runs); 1 MiB chunks force several chunks, a partial last one and
    ring-slot reuse at a size the oracle checks quickly."""
    from paper_1301_4438_b200 import _native

    ctx = _native.context()
    old = ctx.get_option("host_chunk_mb")
    ctx.set_option("host_chunk_mb", 1)
    try:
        a0 = orc.gen_xy_rank(1000, 1100, 700, p, 3)
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(dtype))
        assert a.data.dtype == dtype
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        x = a0.astype(orc.field_dtype(p))
        cc = orc.Counts()
        P, Q, r, _ = orc.pluq(x, p, 30, cc)
        assert f.rank == r and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
        assert np.array_equal(a.data, x) and f.packed is a
        assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == cc.as_tuple()
        # invalid entry in the LAST chunk: EINVAL, buffer untouched
        bad = a0.astype(dtype)
        bad[-1, -1] = p
        keep = bad.copy()
        psig = np.zeros(1000, np.int64); qsig = np.zeros(1100, np.int64); rank = np.zeros(1, np.int64)
        fn = ctx.lib.pluq_factor_host_f64 if dtype == np.float64 else ctx.lib.pluq_factor_host_i64
        st = fn(ctx.handle, bad.ctypes.data, 1000, 1100, p, 30, _native.i64p(psig), _native.i64p(qsig),
                _native.i64p(rank), None)
        assert st == _native.PLUQ_EINVAL and np.array_equal(bad, keep)
    finally:
        ctx.set_option("host_chunk_mb", old)


def test_device_materialization_matches_host(pb):
    """extract_lm / extract_uv / reconstruct / check_structure on a device-resident result
    (matrix.py:308-349) equal the host versions and rebuild A."""
    import torch

    p = 65521
    a0 = orc.gen_xy_rank(300, 260, 170, p, 12)
    fh = pb.pluq(pb.DenseMatrix(pb.PrimeField(p), a0.astype(np.float64)))
    t = torch.from_numpy(a0).cuda().to(torch.int32)
    fd = pb.pluq(pb.DenseMatrix(pb.PrimeField(p), t))
    assert fd.rank == fh.rank == 170
    lm, uv = fd.extract_lm(), fd.extract_uv()
    assert lm.is_cuda and uv.is_cuda
    assert np.array_equal(lm.cpu().numpy().astype(np.int64), fh.extract_lm().astype(np.int64))
    assert np.array_equal(uv.cpu().numpy().astype(np.int64), fh.extract_uv().astype(np.int64))
    rec = fd.reconstruct()
    assert rec.on_device and np.array_equal(rec.data.cpu().numpy().astype(np.int64), a0)
    assert fd.check_structure() == [] == fh.check_structure()


def test_cli_decompose_matches_reference_files(pb, tmp_path):
    """`python -m paper_1301_4438_b200 decompose` writes the reference's own factor file
    (tests/golden/text_fixtures.json), `verify` accepts it, `rank-profile` answers."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "tests", "golden", "text_fixtures.json")) as fh:
        cases = json.load(fh)
    for i, c in enumerate(cases):
        mf = tmp_path / f"m{i}.txt"
        mf.write_text(c["matrix_text"])
        out = subprocess.run([sys.executable, "-m", "paper_1301_4438_b200", "decompose", str(mf)], cwd=root,
                             capture_output=True, text=True)
        assert out.returncode == 0, out.stderr
        assert out.stdout == c["factors_text"], (i, out.stdout, c["factors_text"])
        ff = tmp_path / f"f{i}.txt"
        ff.write_text(out.stdout)
        v = subprocess.run([sys.executable, "-m", "paper_1301_4438_b200", "verify", str(mf), str(ff)], cwd=root,
                           capture_output=True, text=True)
        if not c["factors_readable"]:  # the reference cannot read this file back either (exit 2)
            assert v.returncode == 2
            continue
        assert v.returncode == 0 and v.stdout.strip() == "OK", v.stderr
    rp = subprocess.run([sys.executable, "-m", "paper_1301_4438_b200", "rank-profile", str(tmp_path / "m0.txt")],
                        cwd=root, capture_output=True, text=True)
    assert rp.returncode == 0 and set(json.loads(rp.stdout)) == {"rows", "cols"}


@pytest.mark.parametrize("on_device", [False, True])
def test_to_leu_host_and_device(pb, on_device):
    import torch

    p = 101
    for seed, (m, n, r) in enumerate([(40, 30, 12), (25, 50, 25), (33, 33, 0), (20, 20, 20)]):
        a0 = orc.gen_xy_rank(m, n, r, p, seed) if r else np.zeros((m, n), np.int64)
        orig = pb.DenseMatrix(pb.PrimeField(p), a0.copy())
        data = torch.from_numpy(a0).cuda().to(torch.int32) if on_device else a0.astype(np.float64)
        f = pb.pluq(pb.DenseMatrix(pb.PrimeField(p), data))
        leu = pb.to_leu(f, orig)
        lbar = leu.lbar.host_array()
        e = leu.e.host_array()
        ubar = leu.ubar.host_array()
        assert np.array_equal(np.tril(lbar), lbar) and np.all(np.diagonal(lbar) == 1)
        assert np.array_equal(np.triu(ubar), ubar) and int(e.sum()) == f.rank
        prod = (lbar.astype(object).dot(e.astype(object)).dot(ubar.astype(object))) % p
        assert np.array_equal(prod.astype(np.int64), a0)
        y = np.eye(m - f.rank, dtype=np.int64)
        z = np.zeros((n - f.rank, n - f.rank), np.int64)
        assert pb.check_triangular_extension(f, y, z) == (True, True)


@pytest.mark.parametrize("inplace", [0, 1])
@pytest.mark.parametrize("rows,cols,ld,off,kind", [
    (300, 1000, 1000, 0, "full"),        # every column moves: one staged span per row
    (257, 777, 1031, 3, "full"),         # odd pitch and a misaligned view: scalar head/tail chunks
    (5000, 777, 1031, 1, "full"),        # several rows per CTA: both buffers, odd span
    (3000, 30001, 30001, 0, "full"),     # several rows per CTA, single buffer
    (64, 30000, 30000, 0, "full"),       # span > 100 KB: single buffer
    (40, 60000, 60001, 1, "full"),       # span too wide for shared memory: two-pass path
    (500, 4096, 4100, 2, "window"),      # only columns 1000..3000 move
    (128, 5000, 5000, 0, "sparse"),      # few moved columns over a wide span: two-pass path
    (1, 33, 33, 0, "full"), (700, 2, 2, 0, "full"),
])
def test_permute_cols_paths(pb, rows, cols, ld, off, kind, inplace):
    """apply_cols through the C ABI (matrix.py:267-283 of the reference: X[:, j] <- X[:, g[j]]),
    one-pass in-place gather vs the two-pass path through a temporary, on views with odd
    pitches / offsets."""
    import torch
    from paper_1301_4438_b200 import _native

    rng = np.random.default_rng(rows * 31 + cols)
    g = np.arange(cols)
    if kind == "full":
        g = rng.permutation(cols)
    elif kind == "window":
        g[1000:3000] = 1000 + rng.permutation(2000)
    else:
        idx = rng.choice(cols, 40, replace=False)
        g[np.sort(idx)] = idx
    buf = torch.randint(0, 65521, (rows * ld + off + 8,), dtype=torch.int32, device="cuda")
    before = buf.clone()
    view = buf[off:off + rows * ld].view(rows, ld)
    want = view[:, :cols].cpu().numpy()[:, g]
    ctx = _native.context()
    old = ctx.get_option("gather_inplace")
    ctx.set_option("gather_inplace", inplace)
    try:
        gp = (ctypes.c_int64 * cols)(*g.tolist())
        st = ctx.lib.pluq_permute_cols(ctx.handle, buf.data_ptr() + 4 * off, ld, rows, cols, gp)
        torch.cuda.synchronize()
    finally:
        ctx.set_option("gather_inplace", old)
    assert st == 0
    assert np.array_equal(view[:, :cols].cpu().numpy(), want)
    # nothing outside the view's columns was touched
    mask = torch.ones_like(buf, dtype=torch.bool)
    mask[off:off + rows * ld].view(rows, ld)[:, :cols] = False
    assert torch.equal(buf[mask], before[mask])


@pytest.mark.parametrize("inplace", [0, 1])
@pytest.mark.parametrize("rows,cols,ld,off,moved", [(300, 1000, 1000, 0, 300), (2000, 777, 1031, 3, 40),
                                                    (5000, 4096, 4100, 1, 1536), (5000, 300, 300, 0, 1537),
                                                    (64, 33, 40, 2, 64), (4000, 20000, 20000, 0, 700)])
def test_permute_rows_paths(pb, rows, cols, ld, off, moved, inplace):
    """apply_rows through the C ABI (matrix.py:249-265 of the reference: X[i, :] <- X[g[i], :]),
    one-pass strip gather for small moved sets vs the two-pass path through a temporary."""
    import torch
    from paper_1301_4438_b200 import _native

    rng = np.random.default_rng(rows * 7 + cols)
    g = np.arange(rows)
    idx = np.sort(rng.choice(rows, moved, replace=False))
    g[idx] = rng.permutation(idx)
    buf = torch.randint(0, 65521, (rows * ld + off + 8,), dtype=torch.int32, device="cuda")
    before = buf.clone()
    view = buf[off:off + rows * ld].view(rows, ld)
    want = view[:, :cols].cpu().numpy()[g]
    ctx = _native.context()
    old = ctx.get_option("gather_inplace")
    ctx.set_option("gather_inplace", inplace)
    try:
        gp = (ctypes.c_int64 * rows)(*g.tolist())
        st = ctx.lib.pluq_permute_rows(ctx.handle, buf.data_ptr() + 4 * off, ld, rows, cols, gp)
        torch.cuda.synchronize()
    finally:
        ctx.set_option("gather_inplace", old)
    assert st == 0
    assert np.array_equal(view[:, :cols].cpu().numpy(), want)
    mask = torch.ones_like(buf, dtype=torch.bool)
    mask[off:off + rows * ld].view(rows, ld)[:, :cols] = False
    assert torch.equal(buf[mask], before[mask])


@pytest.mark.parametrize("early", [0, 1])
@pytest.mark.parametrize("kind", ["generic", "rank", "repair", "two_repairs", "fails", "i64"])
def test_host_early_download_vs_oracle(pb, kind, early):
    """Host-buffer pipeline with the early download (option host_early): rows the speculative LU
    announces final are copied back while it still runs (group look-ahead forced on 256-wide
    panels, 1 MiB chunks).  Pivot repairs rotate columns of rows already downloaded (patched
    at the end); a failed speculation invalidates the early chunks.  Bit-exact vs the oracle."""
    from paper_1301_4438_b200 import _native

    p = 8388593 if kind == "i64" else 65521
    dtype = np.int64 if kind == "i64" else np.float64
    m, n = 2600, 2500
    rng = np.random.default_rng(17)
    if kind in ("rank",):
        a0 = np.asarray(orc.gen_xy_rank(m, n, 1800, p, 5), np.int64)
    else:
        a0 = np.asarray(rng.integers(0, p, (m, n)), np.int64)

    def vanish(g, w):
        coef = rng.integers(0, p, g).astype(object)
        a0[g, :g + w] = np.array((coef @ a0[:g, :g + w].astype(object)) % p, dtype=np.int64)

    if kind == "repair":
        vanish(1300, 1)
    if kind == "two_repairs":
        vanish(700, 1); vanish(1900, 2)
    if kind == "fails":  # a row without a pivot deep inside: the speculation fails after many rows were sent
        coef = rng.integers(0, p, 1500).astype(object)
        a0[1500, :] = np.array((coef @ a0[:1500, :].astype(object)) % p, dtype=np.int64)
    x = a0.astype(orc.field_dtype(p))
    cc = orc.Counts()
    P, Q, r, _ = orc.pluq(x, p, 30, cc)
    ctx = _native.context()
    opts = dict(host_chunk_mb=1, host_early=early, small_cap=1, spec_panel=256, la_pair=2, panel_rec=2)
    old = {k: ctx.get_option(k) for k in opts}
    for k, v in opts.items():
        ctx.set_option(k, v)
    try:
        a = pb.DenseMatrix(pb.PrimeField(p), a0.astype(dtype))
        c = pb.OpCounts()
        f = pb.pluq(a, counts=c)
        st = ctx.stats()
    finally:
        for k, v in old.items():
            ctx.set_option(k, v)
    assert f.rank == r and np.array_equal(f.p_perm.sigma, P) and np.array_equal(f.q_perm.sigma, Q)
    assert np.array_equal(a.data, x)
    assert (c.field_mul, c.field_add, c.field_inv, c.modular_reductions) == cc.as_tuple()
    if not early or kind == "fails":
        assert st["early_chunks"] == 0
    # (how many chunks leave early is a matter of timing at this size — the factorization takes
    # ~10 ms; tests/test_gpu_configs.py asserts early_chunks > 0 at cfg5's full size)
