"""Cost of the rare-element drain: each kernel on its config inputs, and on the
same inputs with the drained elements replaced by a typical fast-path argument."""
import sys, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api
L = _lib.ensure_device(0)
for fn, w, dist, n, rep in (("texpm1", 32, "exp32", 1 << 28, 3.0), ("tlog1p", 32, "log32", 1 << 28, 3.0),
                            ("tlog", 32, "log32", 1 << 28, 3.0), ("texpm1", 64, "pow10_64", 1 << 24, 0.25),
                            ("tlog1p", 64, "pow10c_64", 1 << 24, 0.25), ("tlog", 64, "log64", 1 << 26, 3.0)):
    dt = torch.float32 if w == 32 else torch.float64
    x0 = torch.empty(n, dtype=dt, device="cuda"); x1 = torch.empty_like(x0)
    _lib.check(L.tf_generate(_lib.DIST_CODES[dist], 2024, 0, n, x0.data_ptr(), x1.data_ptr(), None), "gen")
    z0 = torch.empty_like(x0); z1 = torch.empty_like(x0)
    lib = api(w)
    def rate(a0, a1):
        for _ in range(3): lib._launch(fn, a0, a1, z0, z1, n, torch.cuda.current_stream().cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): lib._launch(fn, a0, a1, z0, z1, n, torch.cuda.current_stream().cuda_stream)
        e1.record(); torch.cuda.synchronize()
        return n * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    r_cfg = rate(x0, x1)
    # mark drained elements and replace them with a typical fast-path argument
    lib._launch(fn, x0, x1, z0, z1, n, 0, _lib.FLAG_MARK_EXACT); torch.cuda.synchronize()
    rare = z1 == -12345
    y0, y1 = x0.clone(), x1.clone()
    y0[rare] = rep
    y1[rare] = 0.0
    r_clean = rate(y0, y1)
    print(f"{fn} f{w}: drained {rare.float().mean().item():.5f}  cfg {r_cfg:.1f}  without drained elements {r_clean:.1f} G elem/s")
