"""Tensor-core GEMM timing at one shape under the diagnostic modes (option tc_dbg):
0 = normal, 1 = no operand loads after the first ring, 2 = no epilogue, 3 = both."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1301_4438_b200 import _native
m, n, k = (int(v) for v in sys.argv[1:4])
p = 65521
g = torch.Generator().manual_seed(0)
A = torch.randint(0, p, (m, k), generator=g, dtype=torch.int32).cuda()
B = torch.randint(0, p, (k, n), generator=g, dtype=torch.int32).cuda()
C = torch.randint(0, p, (m, n), generator=g, dtype=torch.int32).cuda()
ctx = _native.context()
peak = max(ctx.measure_peaks()["int8_tops"] for _ in range(3))
for opt in sys.argv[4:] or ["tc_dbg=0", "tc_dbg=1", "tc_dbg=2", "tc_dbg=3"]:
    for kv in opt.split(","):
        kk, vv = kv.split("=")
        ctx.set_option(kk, int(vv))
    ctx.set_option("tc_time", 1)
    ts = []
    for it in range(4):
        ctx.lib.pluq_modgemm_sub_tc(ctx.handle, C.data_ptr(), n, A.data_ptr(), k, B.data_ptr(), n, m, n, k, p)
        torch.cuda.synchronize()
        ts.append(ctx.stats()["t_tc_mma_ns"] / 1e6)
    t = min(ts[1:])
    print(f"{m}x{n}x{k} {opt}: mma kernel {t:.3f} ms = {2*m*n*k*4/t/1e9:.0f} TOP/s = {2*m*n*k*4/t/1e9/peak:.3f} of {peak:.0f}", flush=True)
    ctx.set_option("tc_time", 0)
    ctx.set_option("tc_dbg", 0)
