"""Diagnostics run on the GPU box during development (each section isolated)."""
import os, sys, time, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

def sec_tc():
    import torch
    from paper_1301_4438_b200 import _native
    from oracle import pluq_oracle as orc
    ctx = _native.context()
    rng = np.random.default_rng(1)
    for p, (m, n, k) in [(65521, (256, 256, 384)), (65521, (300, 200, 130)), (251, (256, 512, 256)),
                         (8388593, (256, 192, 300)), (2147483647, (128, 128, 128)), (65521, (1024, 1024, 4096))]:
        A = rng.integers(0, p, (m, k)); B = rng.integers(0, p, (k, n)); C = rng.integers(0, p, (m, n))
        tc = torch.from_numpy(C).cuda().to(torch.int32); ta = torch.from_numpy(A).cuda().to(torch.int32); tb = torch.from_numpy(B).cuda().to(torch.int32)
        t0 = time.time()
        st = ctx.lib.pluq_modgemm_sub_tc(ctx.handle, tc.data_ptr(), n, ta.data_ptr(), k, tb.data_ptr(), n, m, n, k, p)
        torch.cuda.synchronize()
        dt = time.time() - t0
        want = orc._mulmod_exact(A, B, p)
        want = (C - want) % p
        got = tc.cpu().numpy().astype(np.int64)
        print(f"tc p={p} {m}x{n}x{k} st={st} ok={np.array_equal(got, want)} mism={(got!=want).sum()} t={dt:.3f}s", flush=True)
        if not np.array_equal(got, want):
            idx = np.argwhere(got != want)[:5]
            print("  first bad", idx.tolist(), [int(got[i,j]) for i,j in idx], [int(want[i,j]) for i,j in idx], flush=True)

def sec_simt():
    import torch
    from paper_1301_4438_b200 import _native
    from oracle import pluq_oracle as orc
    ctx = _native.context(); ctx.set_option("use_tc", 0)
    rng = np.random.default_rng(2)
    for p, (m, n, k) in [(65521, (100, 70, 33)), (8388593, (65, 129, 200)), (2147483647, (40, 50, 60)), (3, (5, 7, 0))]:
        A = rng.integers(0, p, (m, k)); B = rng.integers(0, p, (k, n)); C = rng.integers(0, p, (m, n))
        tc = torch.from_numpy(C).cuda().to(torch.int32); ta = torch.from_numpy(A).cuda().to(torch.int32); tb = torch.from_numpy(B).cuda().to(torch.int32)
        st = ctx.lib.pluq_modgemm_sub(ctx.handle, tc.data_ptr(), n, ta.data_ptr(), max(k,1), tb.data_ptr(), n, m, n, k, p)
        torch.cuda.synchronize()
        want = (C - (orc._mulmod_exact(A, B, p) if k else 0)) % p
        print(f"simt p={p} {m}x{n}x{k} st={st} ok={np.array_equal(tc.cpu().numpy().astype(np.int64), want)}", flush=True)
    ctx.set_option("use_tc", 1)

def sec_golden():
    import paper_1301_4438_b200 as pb
    from paper_1301_4438_b200 import _native
    z = np.load(os.path.join(ROOT, "tests/golden/golden.npz"))
    man = json.load(open(os.path.join(ROOT, "tests/golden/manifest.json")))["cases"]
    import hashlib
    bad = 0; t0 = time.time()
    for e in man:
        k = e["key"]; p = e["p"]
        a = z[k + "_in"]
        field = pb.PrimeField(p)
        A = pb.DenseMatrix(field, a)
        c = pb.OpCounts()
        try:
            f = pb.pluq_iterative(A, c) if e["route"] == "iterative" else pb.pluq(A, threshold=e["threshold"], counts=c)
            ok = (f.rank == e["rank"] and np.array_equal(f.p_perm.sigma, z[k + "_P"]) and np.array_equal(f.q_perm.sigma, z[k + "_Q"])
                  and hashlib.sha256(np.ascontiguousarray(A.data.astype(np.int64)).tobytes()).hexdigest() == e["packed_sha256"]
                  and [c.field_mul, c.field_add, c.field_inv, c.modular_reductions] == e["counts"])
        except Exception as ex:
            ok = False; print("EXC", k, e["tag"], e["route"], e["m"], e["n"], p, repr(ex)[:200], flush=True)
        if not ok:
            bad += 1
            if bad < 8:
                print("BAD", k, e["tag"], e["route"], e["m"], e["n"], p, e["threshold"], flush=True)
    print(f"golden: {bad} bad of {len(man)} in {time.time()-t0:.1f}s", flush=True)

def sec_batch():
    import torch
    import paper_1301_4438_b200 as pb
    from oracle import pluq_oracle as orc
    p = 65521
    batch = orc.gen_cfg2(seed=0, batch=4096)
    t = torch.from_numpy(batch).cuda().to(torch.int32)
    for it in range(3):
        x = t.clone(); torch.cuda.synchronize(); t0 = time.time()
        res = pb.pluq_batched(x, p, 30); torch.cuda.synchronize(); dt = time.time() - t0
    W = 4096 * orc.effective_work(64, 64, 64)
    print(f"batch 4096x64^2: {dt*1e3:.2f} ms  {W/dt/1e9:.1f} Gfield-op/s", flush=True)
    bad = 0
    for b in range(0, 4096, 97):
        xx = batch[b].astype(np.float64); pp, qq, rr, _ = orc.pluq(xx, p, 30)
        if not (int(res.ranks[b]) == rr and np.array_equal(res.p_sigma[b].cpu().numpy(), pp) and np.array_equal(res.packed[b].cpu().numpy(), xx)):
            bad += 1
    print("batch parity bad:", bad, flush=True)

def sec_large():
    import torch
    import paper_1301_4438_b200 as pb
    from oracle import pluq_oracle as orc
    p = 65521
    for n in (512, 2048, 8192):
        a = orc.gen_cfg3(seed=0, n=n) if n != 512 else orc.gen_cfg1(seed=0)
        r_expect = None
        t = torch.from_numpy(a).cuda().to(torch.int32)
        for it in range(2):
            x = t.clone(); A = pb.DenseMatrix(pb.PrimeField(p), x); torch.cuda.synchronize(); t0 = time.time()
            f = pb.pluq(A); torch.cuda.synchronize(); dt = time.time() - t0
        st = pb.last_stats()
        W = orc.effective_work(n, n, f.rank)
        print(f"pluq {n}^2 rank={f.rank} {dt*1e3:.1f} ms {W/dt/1e9:.1f} Gfield-op/s stats={st}", flush=True)
        if n <= 2048:
            ref = a.astype(np.float64); t0 = time.time(); pp, qq, rr, _ = orc.pluq(ref, p, 30); dtc = time.time() - t0
            print(f"   oracle {dtc:.2f}s parity={rr==f.rank and np.array_equal(pp, f.p_perm.sigma) and np.array_equal(x.cpu().numpy(), ref)}", flush=True)

SECS = {"tc": sec_tc, "simt": sec_simt, "golden": sec_golden, "batch": sec_batch, "large": sec_large}
if __name__ == "__main__":
    if len(sys.argv) > 1:
        SECS[sys.argv[1]]()
    else:
        for name in ["simt", "golden", "batch", "tc", "large"]:
            print(f"=== {name}", flush=True)
            r = subprocess.run([sys.executable, __file__, name], timeout=240)
            print(f"=== {name} exit {r.returncode}", flush=True)
