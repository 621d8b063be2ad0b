import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1301_4438_b200 as pb
from paper_1301_4438_b200 import _native
from oracle import pluq_oracle as orc
th = int(sys.argv[1]); nb = int(sys.argv[2])
ctx = _native.context(); ctx.set_option("batch_threads", th)
batch = orc.gen_cfg2(seed=0, batch=nb)
t = torch.from_numpy(batch).cuda().to(torch.int32)
res = pb.pluq_batched(t, 65521, 30); torch.cuda.synchronize()
bad = 0
for b in range(nb):
    x = batch[b].astype(np.float64); P, Q, r, _ = orc.pluq(x, 65521, 30)
    bad += not (int(res.ranks[b]) == r and np.array_equal(t[b].cpu().numpy(), x.astype(np.int64)))
print("threads", th, "bad", bad, "of", nb)
