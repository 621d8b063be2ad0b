"""A/B of the host-buffer path of cfg5 (pluq on a float64 numpy matrix) for an option, alternating
in one process.  usage: python tools/e2e_ab.py option valueA valueB [rounds] [div]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1301_4438_b200 as pb
from paper_1301_4438_b200 import _native, gen
opt, va, vb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
div = int(sys.argv[5]) if len(sys.argv) > 5 else 1
P = 65521
m = 65536 // div
a0 = gen.gen_xy_rank_device(m, m, m // 2, P, seed=0)
host0 = a0.cpu().numpy().astype(np.float64)
del a0
torch.cuda.empty_cache()
buf = np.empty_like(host0)
ctx = _native.context()
ts = {va: [], vb: []}
np.copyto(buf, host0)
dm = pb.DenseMatrix(pb.PrimeField(P), buf)  # validated once, refilled in place per step (as bench.py does)
for r in range(rounds + 1):
    for v in (va, vb):
        ctx.set_option(opt, v)
        np.copyto(buf, host0)
        t0 = time.perf_counter()
        f = pb.pluq(dm)
        dt = time.perf_counter() - t0
        if r:
            ts[v].append(dt)
        print(f"{opt}={v}: {dt*1e3:.0f} ms rank {f.rank} early_chunks {ctx.stats()['early_chunks']}", flush=True)
for v in (va, vb):
    t = sorted(ts[v])
    print(f"{opt}={v}: median {1e3*t[len(t)//2]:.0f} ms min {1e3*t[0]:.0f} max {1e3*t[-1]:.0f}")
