"""Measure pinned H2D / D2H bandwidth and the e2e pipeline pieces."""
import time, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = 1 << 24
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    print(name, f"{n*8/dt/1e9:.1f} GB/s")
t = time.perf_counter()
for _ in range(5):
    z = torch.empty(n, dtype=torch.float64, pin_memory=True)
print("pinned alloc 128MB", (time.perf_counter() - t) / 5 * 1e3, "ms")
from paper_1502_05216_b200 import api, Twofold
f = api(64)
x0 = h.clone().pin_memory(); x0.uniform_(-1, 1); x1 = torch.zeros_like(x0).pin_memory()
f.texpm1(Twofold(x0, x1))
for chunk in (1 << 20, 1 << 22, 1 << 24):
    import paper_1502_05216_b200.explog as E
    t = time.perf_counter()
    for _ in range(3):
        E._pipeline(f, "texpm1", x0, x1, chunk=chunk)
    print("pipeline chunk", chunk, (time.perf_counter() - t) / 3 * 1e3, "ms")
