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
    for kv in os.environ.get("PLUQ_OPTS", "").split(","):
        if kv:
            kk, vv = kv.split("="); _native.context().set_option(kk, int(vv))
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
    if os.environ.get("TC_CFG"): ctx.set_option("tc_cfg", int(os.environ["TC_CFG"]))
    if os.environ.get("TC_GRID"): ctx.set_option("tc_grid", int(os.environ["TC_GRID"]))
    if os.environ.get("TC_DBG"): ctx.set_option("tc_dbg", int(os.environ["TC_DBG"]))
    if os.environ.get("TC_GROUP"): ctx.set_option("tc_group", int(os.environ["TC_GROUP"]))
    if os.environ.get("TC_CPF"): ctx.set_option("tc_cpf", int(os.environ["TC_CPF"]))
    if os.environ.get("TC_VEC"): ctx.set_option("tc_vec", int(os.environ["TC_VEC"]))
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
elif mode == "e2e":
    # transfer anatomy of the host-buffer batched path
    src = orc.gen_cfg2(seed=0, batch=4096).astype(np.float64)
    h = torch.from_numpy(src).pin_memory()
    h2 = torch.empty_like(h).pin_memory()
    d = torch.empty(h.shape, dtype=torch.float64, device="cuda")
    d2 = torch.empty_like(d)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nb = h.numel() * 8
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
        t1 = time.perf_counter(); h2.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize(); t3 = time.perf_counter()
        print(f"h2d {1e3*(t1-t0):.3f} ms ({nb/(t1-t0)/1e9:.1f} GB/s)  d2h {1e3*(t2-t1):.3f} ms "
              f"({nb/(t2-t1)/1e9:.1f} GB/s)  both {1e3*(t3-t2):.3f} ms", flush=True)
    del d, d2
    ctx = _native.context()
    pin = h.numpy()
    for ch in [int(v) for v in sys.argv[2:]] or [8, 4, 16, 32]:
        ctx.set_option("host_chunks", ch)
        for it in range(3):
            pin[...] = src
            torch.cuda.synchronize(); t0 = time.perf_counter()
            r = pb.pluq_batched(pin, P, 30)
            dt = time.perf_counter() - t0
            print(f"e2e chunks={ch}: {1e3*dt:.3f} ms", flush=True)
elif mode == "batchk":
    # per-kernel split of the batched path for option settings given as key=value
    batch = torch.from_numpy(orc.gen_cfg2(seed=0, batch=4096)).cuda().to(torch.int32)
    ctx = _native.context()
    ctx.set_option("time_kernels", 1)
    for spec in sys.argv[2:]:
        for kv in spec.split(","):
            k, v = kv.split("=")
            ctx.set_option(k, int(v))
        for it in range(3):
            x = batch.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
            pb.pluq_batched(x, P, 30); torch.cuda.synchronize()
            st = ctx.stats()
            print(f"{spec}: {1e3*(time.perf_counter()-t0):.3f} ms generic {st['t_generic_ns']/1e3:.1f} us "
                  f"fallback {st['t_fallback_ns']/1e3:.1f} us", flush=True)
elif mode == "e2etrace":
    src = orc.gen_cfg2(seed=0, batch=4096).astype(np.float64)
    h = torch.from_numpy(src).pin_memory(); pin = h.numpy()
    ctx = _native.context()
    for spec in sys.argv[2:] or ["host_chunks=8"]:
        for kv in spec.split(","):
            kk, v = kv.split("="); ctx.set_option(kk, int(v))
        for it in range(3):
            ctx.set_option("trace_pipeline", 1 if it == 2 else 0)
            pin[...] = src
            t0 = time.perf_counter(); r = pb.pluq_batched(pin, P, 30); dt = time.perf_counter() - t0
            ps = np.zeros((4096, 64), np.int64); qs = np.zeros((4096, 64), np.int64); rk = np.zeros(4096, np.int64)
            t1 = time.perf_counter()
            st = ctx.lib.pluq_factor_batched_host_f64(ctx.handle, pin.ctypes.data, 4096, 64, 64, P, 30,
                                                      _native.i64p(ps), _native.i64p(qs), _native.i64p(rk))
            dt2 = time.perf_counter() - t1
            print(f"{spec}: e2e {1e3*dt:.3f} ms  raw C call (reused outputs, already factored input) {1e3*dt2:.3f} ms", flush=True)
    ctx.set_option("trace_pipeline", 0)
elif mode == "cfg5":
    from paper_1301_4438_b200 import gen
    for kv in os.environ.get("PLUQ_OPTS", "").split(","):
        if kv:
            kk, vv = kv.split("="); _native.context().set_option(kk, int(vv))
    div = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    m = 65536 // div; r = 32768 // div
    a0 = gen.gen_xy_rank_device(m, m, r, P, seed=0)
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    x = torch.empty_like(a0)
    for it in range(reps):
        x.copy_(a0); torch.cuda.synchronize()
        last = it == reps - 1 and os.environ.get("PLUQ_PROFILE_LAST")
        if last: torch.cuda.profiler.start()   # ncu --profile-from-start off: only this pluq()
        t0 = time.perf_counter()
        f = pb.pluq(pb.DenseMatrix(pb.PrimeField(P), x)); torch.cuda.synchronize()
        if last: torch.cuda.profiler.stop()
        print(f"cfg5/{div}: {1e3*(time.perf_counter()-t0):.1f} ms rank {f.rank} {pb.last_stats()}", flush=True)
elif mode == "e2emed":
    # median of 10 untraced host-buffer batched calls per option setting
    import statistics
    src = orc.gen_cfg2(seed=0, batch=4096).astype(np.float64)
    h = torch.from_numpy(src).pin_memory(); pin = h.numpy()
    ctx = _native.context()
    for rep in range(2):
        for spec in sys.argv[2:]:
            for kv in spec.split(","):
                kk, v = kv.split("="); ctx.set_option(kk, int(v))
            ts = []
            for it in range(12):
                pin[...] = src
                t0 = time.perf_counter(); r = pb.pluq_batched(pin, P, 30); ts.append(time.perf_counter() - t0)
            print(f"{spec}: e2e median {1e3*statistics.median(ts[2:]):.3f} ms min {1e3*min(ts[2:]):.3f}", flush=True)
elif mode == "cfg4":
    from paper_1301_4438_b200 import gen
    for kv in os.environ.get("PLUQ_OPTS", "").split(","):
        if kv:
            kk, vv = kv.split("="); _native.context().set_option(kk, int(vv))
    div = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    a0, _, _ = gen.gen_cfg4_device(16384 // div, 32768 // div, 8192 // div, 8388593, seed=0)
    for it in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
        x = a0.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
        f = pb.pluq(pb.DenseMatrix(pb.PrimeField(8388593), x)); torch.cuda.synchronize()
        print(f"cfg4/{div}: {1e3*(time.perf_counter()-t0):.1f} ms rank {f.rank} {pb.last_stats()}", flush=True)
