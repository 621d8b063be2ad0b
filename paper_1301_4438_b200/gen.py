"""BASELINE config generators on the SURVEY §8(d) PCG64 stream, products on the device.

SURVEY §8(d) fixes the inputs as ``rng = numpy.random.default_rng(seed)`` (PCG64, the
reference's ``matgen.py:1-7`` convention) with draws in this order:

* cfg1 / cfg5: ``X = rng.integers(0, p, (m, r))``, ``Y = rng.integers(0, p, (r, n))``,
  ``A = X Y mod p``, then ``A = A[rng.permutation(m)][:, rng.permutation(n)]``;
* cfg2: ``rng.integers(0, p, (batch, m, n))``;   cfg3: ``rng.integers(0, p, (n, n))``;
* cfg4: ``I = sort(rng.choice(m, r))``, ``J = sort(rng.choice(n, r))`` (no replacement),
  then X, Y as above with ``X[I_k, k] = 1, X[:I_k, k] = 0, Y[k, J_k] = 1, Y[k, :J_k] = 0``.

The draws here are made by numpy on the host in row chunks and shipped to the device as
int32; the products X Y (K = 8192 / 32768 at cfg4 / cfg5, far beyond what the host can
form) run on the package's own tensor-core modular GEMM.  Two facts make this the SAME
stream as the oracle's single int64 draw (``oracle/pluq_oracle.py:gen_*``), which the
tests check: a bounded draw with range < 2^32 consumes the generator's 32-bit stream
identically for dtype int32 and int64 (numpy's buffered Lemire sampler), and the
generator state carries over between calls, so row chunks concatenate to one draw.
"""

from __future__ import annotations

import numpy as np

from . import _native

# rows per host draw: ~64 MB of int32 per chunk keeps the host footprint bounded at cfg5
_CHUNK_ELEMS = 1 << 24


def _torch():
    import torch

    return torch


def _device(device):
    torch = _torch()
    return device if device is not None else torch.device("cuda", torch.cuda.current_device())


def row_chunks(rng: np.random.Generator, rows: int, cols: int, p: int, chunk_elems: int = _CHUNK_ELEMS):
    """Yield ``(r0, block)``: ``rng.integers(0, p, (rows, cols))`` drawn as int32 row chunks
    (stream-identical to the single int64 draw; pinned by tests/test_gen_stream.py)."""
    step = max(1, chunk_elems // max(1, cols))
    for r0 in range(0, rows, step):
        rc = min(step, rows - r0)
        yield r0, rng.integers(0, p, (rc, cols), dtype=np.int32)


def draw_uniform(rng: np.random.Generator, rows: int, cols: int, p: int, device) -> "object":
    """``rng.integers(0, p, (rows, cols))`` (the int64 stream) as a CUDA int32 tensor."""
    torch = _torch()
    out = torch.empty((rows, cols), dtype=torch.int32, device=device)
    pinned = None
    for r0, blk in row_chunks(rng, rows, cols, p):
        rc = blk.shape[0]
        if pinned is None or pinned.shape[0] < rc:
            pinned = torch.empty((rc, cols), dtype=torch.int32, pin_memory=True)
        pinned[:rc].numpy()[...] = blk
        out[r0:r0 + rc].copy_(pinned[:rc])
    return out


def device_matmul_mod_t(x, y, p: int):
    """X Y mod p for CUDA int32 tensors (exact, tensor-core GEMM for large shapes)."""
    torch = _torch()
    m, k = x.shape
    n = y.shape[1]
    c = torch.zeros((m, n), dtype=torch.int32, device=x.device)
    if m == 0 or n == 0 or k == 0:
        return c
    x = x.contiguous()
    y = y.contiguous()
    ctx = _native.context(x.device.index)
    st = ctx.lib.pluq_modgemm_sub(ctx.handle, c.data_ptr(), n, x.data_ptr(), k, y.data_ptr(), n, m, n, k, p)
    _native.raise_for(st, ctx, "generator gemm")
    # c = -XY mod p  ->  XY mod p, in place
    c.neg_().add_(p)
    c.masked_fill_(c == p, 0)
    return c


def _permute(a, rp: np.ndarray, cp: np.ndarray):
    """a[rp][:, cp] on the device, one full-size temporary at a time."""
    torch = _torch()
    dev = a.device
    a = torch.index_select(a, 0, torch.from_numpy(rp).to(dev))
    return torch.index_select(a, 1, torch.from_numpy(cp).to(dev))


def gen_xy_rank_device(m: int, n: int, r: int, p: int, seed: int = 0, permute: bool = True, device=None):
    """cfg1 / cfg5 family; equals ``oracle.gen_xy_rank(m, n, r, p, seed)``."""
    dev = _device(device)
    rng = np.random.default_rng(seed)
    x = draw_uniform(rng, m, r, p, dev)
    y = draw_uniform(rng, r, n, p, dev)
    a = device_matmul_mod_t(x, y, p)
    del x, y
    if permute:
        rp = rng.permutation(m)
        cp = rng.permutation(n)
        a = _permute(a, rp, cp).contiguous()
    return a


def gen_cfg1_device(seed: int = 0, device=None):
    return gen_xy_rank_device(512, 512, 384, 65521, seed, device=device)


def gen_cfg5_device(seed: int = 0, n: int = 65536, r: int = 32768, p: int = 65521, device=None):
    return gen_xy_rank_device(n, n, r, p, seed, device=device)


def gen_cfg2_device(seed: int = 0, batch: int = 4096, m: int = 64, n: int = 64, p: int = 65521, device=None):
    """cfg2: ``rng.integers(0, p, (batch, m, n))`` as a CUDA int32 (batch, m, n) tensor."""
    dev = _device(device)
    rng = np.random.default_rng(seed)
    return draw_uniform(rng, batch * m, n, p, dev).view(batch, m, n)


def gen_cfg3_device(seed: int = 0, n: int = 8192, p: int = 65521, device=None):
    dev = _device(device)
    return draw_uniform(np.random.default_rng(seed), n, n, p, dev)


def gen_cfg4_device(m: int = 16384, n: int = 32768, r: int = 8192, p: int = 8388593, seed: int = 0, device=None):
    """cfg4: prescribed rank profiles (I, J); equals ``oracle.gen_cfg4``.  Returns (A, I, J)."""
    torch = _torch()
    dev = _device(device)
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(m, r, replace=False))
    cols = np.sort(rng.choice(n, r, replace=False))
    x = draw_uniform(rng, m, r, p, dev)
    y = draw_uniform(rng, r, n, p, dev)
    ti = torch.from_numpy(rows).to(dev)
    tj = torch.from_numpy(cols).to(dev)
    kk = torch.arange(r, device=dev)
    x.masked_fill_(torch.arange(m, device=dev)[:, None] < ti[None, :], 0)
    x[ti, kk] = 1
    y.masked_fill_(torch.arange(n, device=dev)[None, :] < tj[:, None], 0)
    y[kk, tj] = 1
    a = device_matmul_mod_t(x, y, p)
    return a, rows, cols
