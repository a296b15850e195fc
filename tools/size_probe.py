"""Kernel time vs element count and input mix (fixed overhead / tail probe)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1502_05216_b200 import _lib, api  # noqa: E402

L = _lib.ensure_device(0)
dev = torch.device("cuda", 0)
lib = api(64)


def timeit(fn, a0, a1, reps=20):
    z0, z1 = torch.empty_like(a0), torch.empty_like(a0)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        lib._launch(fn, a0, a1, z0, z1, a0.numel(), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib._launch(fn, a0, a1, z0, z1, a0.numel(), s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for fn, dist in (("texpm1", 1), ("tlog1p", 2)):
    for n in [1 << k for k in (12, 16, 18, 20, 21, 22, 24, 26)]:
        a0 = torch.empty(n, dtype=torch.float64, device=dev)
        a1 = torch.empty_like(a0)
        _lib.check(L.tf_generate(dist, 2024, 0, n, a0.data_ptr(), a1.data_ptr(), None), "gen")
        t_cfg = timeit(fn, a0, a1)
        c0 = (torch.rand(n, dtype=torch.float64, device=dev) - 0.5) * 0.6
        c1 = c0 * (torch.rand_like(c0) - 0.5) * 2.0 ** -53
        t_clean = timeit(fn, c0, c1)
        cnt = torch.zeros(1, dtype=torch.int64)
        print(f"{fn} n=2^{n.bit_length()-1}: cfg {t_cfg*1e3:8.1f} us ({n/t_cfg/1e6:6.1f} G/s)  "
              f"clean {t_clean*1e3:8.1f} us ({n/t_clean/1e6:6.1f} G/s)", flush=True)
