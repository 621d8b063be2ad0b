"""Dev sweep of driver knobs on the GPU box (not part of the product)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1301_4438_b200 as pb
from paper_1301_4438_b200 import _native
from oracle import pluq_oracle as orc
P = 65521
ctx = _native.context()
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "batch"):
    batch = torch.from_numpy(orc.gen_cfg2(seed=0, batch=4096)).cuda().to(torch.int32)
    for th in (32, 64, 128, 256):
        ctx.set_option("batch_threads", th)
        ts = []
        for it in range(4):
            x = batch.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
            pb.pluq_batched(x, P, 30); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        W = 4096 * orc.effective_work(64, 64, 64)
        print(f"batch threads={th}: {min(ts)*1e3:.3f} ms  {W/min(ts)/1e9:.1f} Gfop/s", flush=True)
if what in ("all", "cfg3"):
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    a = torch.from_numpy(orc.gen_cfg3(seed=0, n=n)).cuda().to(torch.int32)
    for cap in (32 * 32, 64 * 64, 128 * 128):
        for th in (32, 64, 128, 256):
            ctx.set_option("small_cap", cap); ctx.set_option("small_threads", th)
            ts = []
            for it in range(2):
                x = a.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
                f = pb.pluq(pb.DenseMatrix(pb.PrimeField(P), x)); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
            print(f"cfg3 n={n} cap={cap} threads={th}: {min(ts)*1e3:.1f} ms rank={f.rank} {orc.effective_work(n,n,f.rank)/min(ts)/1e9:.0f} Gfop/s {pb.last_stats()}", flush=True)
    ctx.set_option("small_cap", 128 * 128); ctx.set_option("small_threads", 256)
