"""PCIe floor of the host-buffer batch pipeline: cfg2-sized float64 H2D copies chained to
D2H copies chunk by chunk (no kernels), for several chunk counts."""
import torch, time
n = 4096*64*64
h = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for C in (1, 8, 24, 64):
    ts = []
    for it in range(6):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        step = (n + C - 1) // C
        evs = []
        for k in range(C):
            a, b = k * step, min(n, (k + 1) * step)
            with torch.cuda.stream(s1):
                d[a:b].copy_(h[a:b], non_blocking=True); e = torch.cuda.Event(); e.record(s1)
            s2.wait_event(e)
            with torch.cuda.stream(s2):
                h2[a:b].copy_(d[a:b], non_blocking=True)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(f"chunks {C}: H2D->D2H chained copies {1e3*sorted(ts)[2]:.3f} ms", flush=True)
