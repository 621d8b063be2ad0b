"""A/B of a tensor-core GEMM option inside one process (alternating, so both see the same thermal state).
usage: python tools/gemm_ab.py M N K option valueA valueB [rounds]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1301_4438_b200 import _native
m, n, k = (int(v) for v in sys.argv[1:4])
opt, va, vb = sys.argv[4], int(sys.argv[5]), int(sys.argv[6])
rounds = int(sys.argv[7]) if len(sys.argv) > 7 else 6
p = 65521
g = torch.Generator().manual_seed(0)
A = torch.randint(0, p, (m, k), generator=g, dtype=torch.int32).cuda()
B = torch.randint(0, p, (k, n), generator=g, dtype=torch.int32).cuda()
C = torch.randint(0, p, (m, n), generator=g, dtype=torch.int32).cuda()
ctx = _native.context()
ts = {va: [], vb: []}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(rounds + 1):
    for v in (va, vb):
        ctx.set_option(opt, v)
        torch.cuda.synchronize(); e0.record()
        st = ctx.lib.pluq_modgemm_sub_tc(ctx.handle, C.data_ptr(), n, A.data_ptr(), k, B.data_ptr(), n, m, n, k, p)
        e1.record(); torch.cuda.synchronize()
        if r: ts[v].append(e0.elapsed_time(e1))
for v in (va, vb):
    t = sorted(ts[v])
    print(f"{m}x{n}x{k} {opt}={v}: median {t[len(t)//2]:.3f} ms min {t[0]:.3f} max {t[-1]:.3f}  ({2*m*n*k/t[len(t)//2]/1e9:.1f} Tfop/s)")
