"""Pinned host<->device copies of the cfg2 state (50 MB) cut into chunks, on one or
two streams per direction, both directions concurrently (adg_step_host's copy pattern
without the sweep dependencies)."""
import torch, time, sys
n = 50388480 // 8
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True); h2 = torch.empty_like(h1).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty_like(d1)
si = [torch.cuda.Stream() for _ in range(2)]; so = [torch.cuda.Stream() for _ in range(2)]
def t(f, k=10):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
def chunked(c, ns, inplace=False):
    b = [n * i // c for i in range(c + 1)]
    hd = h1 if inplace else h2
    def f():
        for i in range(c):
            with torch.cuda.stream(si[i % ns]): d1[b[i]:b[i+1]].copy_(h1[b[i]:b[i+1]], non_blocking=True)
            with torch.cuda.stream(so[i % ns]): hd[b[i]:b[i+1]].copy_(d2[b[i]:b[i+1]], non_blocking=True)
    return f
for c in (1, 8, 16, 23, 32):
    for ns in (1, 2):
        print("chunks %2d streams/dir %d: both %.3f ms  (same host buffer %.3f ms)"
              % (c, ns, t(chunked(c, ns)), t(chunked(c, ns, True))))
