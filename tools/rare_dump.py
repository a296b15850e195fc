"""Dump inputs that the fast band rejects (TF_FLAG_MARK_EXACT) per config."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api, workloads
n = 1 << 20
res = {}
for cfg, (fn, w, dist, _) in workloads.CONFIGS.items():
    x0, x1 = workloads.generate(dist, 0, n, seed=1)
    t0 = torch.from_numpy(x0).cuda(); t1 = torch.from_numpy(x1).cuda()
    z = api(w)._device(fn, t0, t1, flags=_lib.FLAG_MARK_EXACT)
    z1 = z.error.cpu().numpy()
    idx = np.nonzero(z1 == -12345)[0]
    res[cfg] = idx
    print(cfg, len(idx) / n)
np.savez_compressed("gpurun_out/rare.npz", **res)
