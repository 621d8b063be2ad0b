"""N>1 host logic on CPU: world_size-2 gloo process group (batch sharding has no
data-path collective; only timing/work reduction and an optional rank gather)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1301_4438_b200.sharding import gather_ranks, reduce_timing, shard_range, shard_seed


def test_shard_range_partitions():
    for total in (0, 1, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
    assert shard_seed(5, 3) == 8


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle import pluq_oracle as orc

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        total, p = 12, 101
        batch = orc.gen_cfg2(seed=0, batch=total, m=10, n=10, p=p)
        batch[3] = 0
        batch[7] = np.outer(np.arange(10), np.arange(10)) % p
        lo, hi = shard_range(total, rank, world)
        ranks = []
        for b in range(lo, hi):
            x = batch[b].astype(np.float64)
            _, _, r, _ = orc.pluq(x, p, 30)  # stand-in for the device kernel on this rank
            ranks.append(r)
        t, w = reduce_timing(0.5 + rank, float(hi - lo))
        allr = gather_ranks(np.array(ranks), total)
        q.put((rank, t, w, allr.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    from oracle import pluq_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    total, p = 12, 101
    batch = orc.gen_cfg2(seed=0, batch=total, m=10, n=10, p=p)
    batch[3] = 0
    batch[7] = np.outer(np.arange(10), np.arange(10)) % p
    want = [orc.pluq(batch[b].astype(np.float64), p, 30)[2] for b in range(total)]
    for rank, t, w, allr in res:
        assert t == 1.5          # max over ranks of 0.5 + rank
        assert w == float(total)  # every matrix counted exactly once
        assert allr == want
