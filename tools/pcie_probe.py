"""Measure pinned H2D / D2H bandwidth (each alone and both at once), the host
pipeline at several chunk sizes, and a zero-copy launch (the kernel reading
and writing pinned host memory directly)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = 1 << 24
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def bw(name, fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"{name:28s} {nbytes / dt / 1e9:7.1f} GB/s")


def both():
    with torch.cuda.stream(sa):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(sb):
        h2.copy_(d2, non_blocking=True)


bw("h2d", lambda: d.copy_(h, non_blocking=True), n * 8)
bw("d2h", lambda: h.copy_(d, non_blocking=True), n * 8)
bw("h2d+d2h concurrent (sum)", both, 2 * n * 8)

import paper_1502_05216_b200.explog as E  # noqa: E402
from paper_1502_05216_b200 import Twofold, api  # noqa: E402

f = api(64)
x0 = torch.empty(n, dtype=torch.float64).uniform_(-1, 1).pin_memory()
x1 = torch.zeros_like(x0).pin_memory()
o0, o1 = torch.empty_like(x0).pin_memory(), torch.empty_like(x0).pin_memory()
ref = f.texpm1(Twofold(x0.cuda(), x1.cuda()))
r0, r1 = ref.value.cpu(), ref.error.cpu()
for chunk in (1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22, 1 << 23):
    E._pipeline(f, "texpm1", x0, x1, chunk=chunk, out=(o0, o1))
    t = time.perf_counter()
    for _ in range(5):
        E._pipeline(f, "texpm1", x0, x1, chunk=chunk, out=(o0, o1))
    dt = (time.perf_counter() - t) / 5
    ok = torch.equal(o0, r0) and torch.equal(o1, r1)
    print(f"pipeline chunk 2^{chunk.bit_length() - 1}: {dt * 1e3:7.2f} ms "
          f"{n / dt / 1e9:6.2f} G elem/s ({4 * n * 8 / dt / 1e9:6.1f} GB/s both ways) ok={ok}")

# zero-copy measured 14 GB/s both ways (cp.async staging from sysmem): off by default
if os.environ.get("ZERO_COPY", "0") == "1":
    from paper_1502_05216_b200 import _lib  # noqa: E402

    s = torch.cuda.current_stream().cuda_stream
    o0.zero_()
    o1.zero_()
    L = _lib.ensure_device(0)

    def zc():
        rc = L.tf_eval(_lib.FN_CODES["texpm1"], 64, x0.data_ptr(), x1.data_ptr(),
                       o0.data_ptr(), o1.data_ptr(), n, s, 0)
        _lib.check(rc, "zero-copy tf_eval")

    zc()
    torch.cuda.synchronize()
    ok = torch.equal(o0, r0) and torch.equal(o1, r1)
    t = time.perf_counter()
    for _ in range(5):
        zc()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"zero-copy kernel: {dt * 1e3:7.2f} ms {n / dt / 1e9:6.2f} G elem/s "
          f"({4 * n * 8 / dt / 1e9:6.1f} GB/s both ways) ok={ok}")
