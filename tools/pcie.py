"""PCIe bandwidth on the box: H2D, D2H and both concurrently, 2 GiB pinned (development tool)."""
import time
import torch
n = 2 * 2**30 // 16
h1 = torch.empty(n, dtype=torch.complex128).pin_memory()
h2 = torch.empty(n, dtype=torch.complex128).pin_memory()
d1 = torch.empty(n, dtype=torch.complex128, device="cuda")
d2 = torch.empty(n, dtype=torch.complex128, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for label, fn in [("h2d", lambda: d1.copy_(h1, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(label, "%.1f GB/s" % (n * 16 / dt / 1e9))
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("both", "%.1f GB/s each, %.1f ms" % (n * 16 / dt / 1e9, dt * 1e3))
