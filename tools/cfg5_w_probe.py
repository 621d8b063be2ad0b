"""cfg5 with a given outer panel width: time, stats, and a device Freivalds check."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1301_4438_b200 as pb
from paper_1301_4438_b200 import _native, gen, verify
ctx = _native.context()
a0 = gen.gen_cfg5_device(seed=0)
for spec in sys.argv[1:]:
    for kv in spec.split(","):
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    x = a0.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
    f = pb.pluq(pb.DenseMatrix(pb.PrimeField(65521), x)); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = pb.last_stats()
    print(f"{spec}: {dt*1e3:.1f} ms rank {f.rank} spec_ok {st['speculative_ok']} fail {st['speculative_fail']} "
          f"repairs {st['spec_repairs']} freivalds {verify.freivalds(a0, f, probes=1)}", flush=True)
    del x, f
