"""One large matrix across N GPUs (paper_1301_4438_b200.distributed), timed as the max over
ranks of device-synchronised wall time.  Launch:
  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
      --master-port 29531 tools/dist_single.py cfg3|cfg5 [div] [panel] [pr]
(cfg5 = 65536^2 rank 32768 / div; cfg3 = 8192^2 / div; pr > 0 selects the 2D pr x (N/pr)
grid, the default is the 1 x N column-panel layout).  Rank 0 checks rank, structure and
Freivalds.  Single process without torchrun: world size 1."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import torch.distributed as dist

import paper_1301_4438_b200 as pb
from paper_1301_4438_b200 import gen, verify
from paper_1301_4438_b200.sharding import reduce_timing

which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
div = int(sys.argv[2]) if len(sys.argv) > 2 else 1
width = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
prow = int(sys.argv[4]) if len(sys.argv) > 4 else 0
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl")
p = 65521
if which == "cfg5":
    m = n = 65536 // div
    a0 = gen.gen_xy_rank_device(m, n, 32768 // div, p, seed=0) if rank == 0 else None
else:
    m = n = 8192 // div
    g = torch.Generator(device="cuda").manual_seed(0)
    a0 = torch.randint(0, p, (m, n), generator=g, device="cuda", dtype=torch.int64).to(torch.int32) if rank == 0 else None
for it in range(2):
    a = pb.DenseMatrix(pb.PrimeField(p), a0.clone()) if rank == 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = pb.pluq_distributed(a, m, n, p, 30, width=width, grid=(prow, world // prow) if prow else None)
    torch.cuda.synchronize()
    t, _ = reduce_timing(time.perf_counter() - t0, 0.0, torch.device("cuda", local))
    if rank == 0:
        r = f.rank
        W = 2.0 * m * n * r - (m + n) * float(r) ** 2 + 2.0 * float(r) ** 3 / 3.0
        print(f"{which}/{div} on {world} GPU(s): {t*1e3:.1f} ms rank {r} {W/t/1e9:.1f} Gfield-op/s", flush=True)
if rank == 0:
    print("structure", verify.structure_ok(f), "freivalds", verify.freivalds(a0, f, probes=2), flush=True)
if world > 1:
    dist.destroy_process_group()
