"""Pinned host<->device copy bandwidth alone and concurrent (50 MB, the cfg2 state)."""
import torch, time
n = 50388480 // 8
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True); h2 = torch.empty_like(h1).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty_like(d1)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, k=10):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("h2d ms %.3f  d2h ms %.3f  both ms %.3f" % (t(lambda: d1.copy_(h1, non_blocking=True)),
      t(lambda: h2.copy_(d2, non_blocking=True)), t(both)))
