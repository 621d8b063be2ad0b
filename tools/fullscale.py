"""Full-scale BASELINE configs on one B200 with property checks (rank, profiles,
structure, Freivalds).  Usage: python tools/fullscale.py cfg3|cfg4|cfg5 [scale_div]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1301_4438_b200 as pb
from paper_1301_4438_b200 import gen, verify


def work(m, n, r):
    return 2.0 * m * n * r - (m + n) * float(r) ** 2 + 2.0 * float(r) ** 3 / 3.0


which = sys.argv[1]
div = int(sys.argv[2]) if len(sys.argv) > 2 else 1
torch.cuda.set_device(0)
t0 = time.perf_counter()
if which == "cfg4":
    m, n, r, p = 16384 // div, 32768 // div, 8192 // div, 8388593
    a, rows, cols = gen.gen_cfg4_device(m, n, r, p, seed=0)
elif which == "cfg5":
    m = n = 65536 // div
    r, p = 32768 // div, 65521
    a = gen.gen_xy_rank_device(m, n, r, p, seed=0)
    rows = cols = None
else:
    m = n = 8192 // div
    p = 65521
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randint(0, p, (m, n), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
    rows = cols = None
torch.cuda.synchronize()
print(f"{which}: generated {m}x{n} on device in {time.perf_counter()-t0:.2f}s", flush=True)
orig = a.clone()
times = []
for it in range(2):
    x = orig.clone()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = pb.pluq(pb.DenseMatrix(pb.PrimeField(p), x))
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t0)
    print(f"  run {it}: {times[-1]*1e3:.1f} ms rank {f.rank} stats {pb.last_stats()}", flush=True)
r_got = f.rank
W = work(m, n, r_got)
print(f"{which}: rank={r_got} best={min(times)*1e3:.1f} ms  W={W:.3e}  {W/min(times)/1e9:.1f} Gfield-op/s", flush=True)
ok = verify.structure_ok(f)
fr = verify.freivalds(orig, f, probes=2)
line = f"{which}: structure_ok={ok} freivalds={fr}"
if rows is not None:
    line += f" row_profile_ok={pb.row_rank_profile(f) == tuple(int(v) for v in rows)}"
    line += f" col_profile_ok={pb.col_rank_profile(f) == tuple(int(v) for v in cols)}"
print(line, flush=True)
