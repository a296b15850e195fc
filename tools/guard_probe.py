"""Fast path vs forced exact path on large config samples: z0 / z1 bit mismatches.
Run against a library built with a tight rounding guard (e.g. -DTF_TOL32_LOG=-40)
to bound the binary32 cores' value-part error empirically.
usage: python tools/guard_probe.py [log2 n] [seeds] [width]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api
L = _lib.ensure_device(0)
n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 26)
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = int(sys.argv[3]) if len(sys.argv) > 3 else 32
cases = ((("texp", "exp32"), ("texpm1", "exp32"), ("tlog", "log32"), ("tlog1p", "log32")) if w == 32
         else (("texp", "exp64"), ("texpm1", "pow10_64"), ("tlog", "log64"), ("tlog1p", "pow10c_64")))
iv = torch.int32 if w == 32 else torch.int64
for fn, dist in cases:
    x0 = torch.empty(n, dtype=torch.float32 if w == 32 else torch.float64, device="cuda")
    x1 = torch.empty_like(x0)
    za, zb, ea, eb = (torch.empty_like(x0) for _ in range(4))
    m0 = m1 = 0
    for seed in range(seeds):
        _lib.check(L.tf_generate(_lib.DIST_CODES[dist], 7000 + seed, 0, n, x0.data_ptr(), x1.data_ptr(), None), "gen")
        api(w)._launch(fn, x0, x1, za, zb, n, 0, 0)
        api(w)._launch(fn, x0, x1, ea, eb, n, 0, _lib.FLAG_FORCE_EXACT)
        torch.cuda.synchronize()
        bad = (za.view(iv) != ea.view(iv)).nonzero().flatten()[:4].tolist()
        for i in bad:
            print(f"  {fn} seed {seed} i {i}: x = ({x0[i].item().hex()}, {x1[i].item().hex()}) "
                  f"fast z0 {za[i].item().hex()} exact z0 {ea[i].item().hex()}")
        m0 += int((za.view(iv) != ea.view(iv)).sum())
        m1 += int((zb.view(iv) != eb.view(iv)).sum())
    print(f"{fn:7s} f{w} {seeds} x 2^{n.bit_length() - 1}: z0 mismatches {m0}, z1 mismatches {m1}")
