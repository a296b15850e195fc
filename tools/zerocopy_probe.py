"""End-to-end host-array evaluation: tf_eval_host's copy-engine chunk pipeline
against one kernel launch on the pinned host buffers themselves (zero-copy: the
kernel's cp.async loads and streaming stores cross PCIe directly).

    python tools/zerocopy_probe.py [log2 n]      (GPU box)
"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib  # noqa: E402

L = _lib.ensure_device(0)
n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 28)
sp = torch.cuda.current_stream().cuda_stream
res = {}
for fn, dist in (("texp", "exp64s"), ("tlog", "logu64s")):
    d0 = torch.empty(n, dtype=torch.float64, device="cuda")
    d1 = torch.empty_like(d0)
    _lib.check(L.tf_generate(_lib.DIST_CODES[dist], 2024, 0, n, d0.data_ptr(), d1.data_ptr(), sp),
               "gen")
    h0 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h0.copy_(d0)
    h1.copy_(d1)
    ref0, ref1 = torch.empty_like(d0), torch.empty_like(d0)
    code = _lib.FN_CODES[fn]
    _lib.check(L.tf_eval(code, 64, d0.data_ptr(), d1.data_ptr(), ref0.data_ptr(), ref1.data_ptr(),
                         n, sp, 0), "ref")
    del d0, d1
    o0 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    o1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()

    def pipe():
        _lib.check(L.tf_eval_host(code, 64, h0.data_ptr(), h1.data_ptr(), o0.data_ptr(),
                                  o1.data_ptr(), n, 0, None, 0), "host")

    def zc():
        _lib.check(L.tf_eval(code, 64, h0.data_ptr(), h1.data_ptr(), o0.data_ptr(), o1.data_ptr(),
                             n, sp, 0), "zc")
        torch.cuda.synchronize()

    for name, f in (("pipeline", pipe), ("zerocopy", zc)):
        f()
        t = time.perf_counter()
        for _ in range(3):
            f()
        dt = (time.perf_counter() - t) / 3
        same = torch.equal(o0.cuda().view(torch.int64), ref0.view(torch.int64)) and \
            torch.equal(o1.cuda().view(torch.int64), ref1.view(torch.int64))
        res[f"{fn}_{name}"] = (round(n / dt / 1e9, 3), round(32 * n / dt / 1e9, 1), same)
        print(fn, name, f"{n / dt / 1e9:.3f} G elem/s", f"{32 * n / dt / 1e9:.1f} GB/s both ways",
              "bit-equal" if same else "DIFFERENT", flush=True)
    del h0, h1, o0, o1, ref0, ref1
    torch.cuda.empty_cache()
