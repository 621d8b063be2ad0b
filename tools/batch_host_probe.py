import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1301_4438_b200 as pb
from oracle import pluq_oracle as orc
P = 65521
batch = torch.from_numpy(orc.gen_cfg2(seed=0, batch=4096)).cuda().to(torch.int32)
xs = [batch.clone() for _ in range(40)]
for x in xs[:5]: pb.pluq_batched(x, P, 30)
torch.cuda.synchronize()
t0 = time.perf_counter()
for x in xs[5:25]: r = pb.pluq_batched(x, P, 30)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"20 calls: host enqueue {1e3*(t1-t0)/20:.3f} ms/call, total {1e3*(t2-t0)/20:.3f} ms/call")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for x in xs[25:35]: r = pb.pluq_batched(x, P, 30)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats('cumulative').print_stats(14)
