"""Where does the seed-0 cfg5 input leave the generic rank profile?  (diagnostic)"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1301_4438_b200 as pb
from paper_1301_4438_b200 import gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
a0 = gen.gen_xy_rank_device(n, n, n // 2, 65521, seed=seed)
x = a0.clone()
torch.cuda.synchronize(); t0 = time.perf_counter()
f = pb.pluq(pb.DenseMatrix(pb.PrimeField(65521), x)); torch.cuda.synchronize()
dt = time.perf_counter() - t0
P, Q = f.p_perm.sigma, f.q_perm.sigma
badp = np.nonzero(P != np.arange(n))[0]
badq = np.nonzero(Q != np.arange(n))[0]
print(f"n={n} seed={seed} rank={f.rank} time={dt:.3f}s stats={pb.last_stats()}")
print("P non-fixed:", len(badp), badp[:20], P[badp[:20]])
print("Q non-fixed:", len(badq), badq[:20], Q[badq[:20]])
rows = pb.row_rank_profile(f); cols = pb.col_rank_profile(f)
rr = np.array(rows); cc = np.array(cols)
print("row profile != 0..r-1 at", np.nonzero(rr != np.arange(len(rr)))[0][:10], "col at", np.nonzero(cc != np.arange(len(cc)))[0][:10])
pairs = [(int(np.argsort(P)[t]), int(Q[t])) for t in range(f.rank)]
off = [(t, pq) for t, pq in enumerate(pairs) if pq[0] != pq[1]]
print("off-diagonal support pairs:", len(off), off[:20])
