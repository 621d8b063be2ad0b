"""Run one workload once (for ncu launch lists / profiling on the GPU box)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1301_4438_b200 as pb
from paper_1301_4438_b200 import _native
from oracle import pluq_oracle as orc
P = 65521
mode = sys.argv[1]
if mode == "cfg3":
    n = int(sys.argv[2])
    a = torch.from_numpy(orc.gen_cfg3(seed=0, n=n)).cuda().to(torch.int32)
    for it in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
        x = a.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
        f = pb.pluq(pb.DenseMatrix(pb.PrimeField(P), x)); torch.cuda.synchronize()
        print(f"cfg3 {n}: {1e3*(time.perf_counter()-t0):.1f} ms rank {f.rank} {pb.last_stats()}", flush=True)
elif mode == "gemm":
    m, n, k = (int(v) for v in sys.argv[2:5])
    p = int(sys.argv[5]) if len(sys.argv) > 5 else P
    g = torch.Generator().manual_seed(0)
    A = torch.randint(0, p, (m, k), generator=g, dtype=torch.int32).cuda()
    B = torch.randint(0, p, (k, n), generator=g, dtype=torch.int32).cuda()
    C = torch.randint(0, p, (m, n), generator=g, dtype=torch.int32).cuda()
    ctx = _native.context()
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = ctx.lib.pluq_modgemm_sub_tc(ctx.handle, C.data_ptr(), n, A.data_ptr(), k, B.data_ptr(), n, m, n, k, p)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"gemm {m}x{n}x{k} p={p}: st={st} {dt*1e3:.3f} ms {2*m*n*k/dt/1e12:.1f} Tfop/s", flush=True)
elif mode == "batch":
    batch = torch.from_numpy(orc.gen_cfg2(seed=0, batch=4096)).cuda().to(torch.int32)
    for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
        x = batch.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
        pb.pluq_batched(x, P, 30); torch.cuda.synchronize()
        print(f"batch: {1e3*(time.perf_counter()-t0):.3f} ms", flush=True)
