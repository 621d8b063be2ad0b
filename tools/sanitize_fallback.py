"""Stress check of the generic -> rank-profile hand-off (prefix slots, streaming consumer
when the batch has >= 1024 blocks): a batch with non-generic 64x64 blocks (early, late and
rank-deficient failures) checked against the oracle.  usage: sanitize_fallback.py BATCH"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1301_4438_b200 as pb
from oracle import pluq_oracle as orc

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 160
p = 65521
rng = np.random.default_rng(7)
batch = rng.integers(0, p, (nb, 64, 64))
bad_idx = rng.choice(nb, min(nb, 24), replace=False)
for k, b in enumerate(bad_idx):
    if k % 3 == 0:
        batch[b] = orc.gen_xy_rank(64, 64, 63, p, int(b))      # fails at the last pivot
    elif k % 3 == 1:
        batch[b] = orc.gen_xy_rank(64, 64, int(rng.integers(1, 63)), p, int(b))
    else:
        batch[b][:, int(rng.integers(0, 40))] = 0                 # zero column
t = torch.from_numpy(batch).cuda().to(torch.int32)
res = pb.pluq_batched(t, p, 30)
torch.cuda.synchronize()
check = sorted(set(bad_idx.tolist()) | set(range(0, nb, max(1, nb // 16))))
bad = 0
for b in check:
    x = batch[b].astype(orc.field_dtype(p))
    P, Q, r, _ = orc.pluq(x, p, 30)
    bad += not (int(res.ranks[b]) == r and np.array_equal(res.p_sigma[b].cpu().numpy(), P)
                and np.array_equal(t[b].cpu().numpy(), x.astype(np.int64)))
print(f"batch {nb}: {len(check)} blocks checked against the oracle, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
