"""Print golden inputs where the fast kernel and the forced exact path differ."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1502_05216_b200 import _lib, api  # noqa: E402

fn, width = sys.argv[1], int(sys.argv[2])
g = np.load(f"tests/golden/golden_{fn}_f{width}.npz")
dev = torch.device("cuda", 0)
x0 = torch.from_numpy(g["x0"]).to(dev)
x1 = torch.from_numpy(g["x1"]).to(dev)
lib = api(width)
a = lib._device(fn, x0, x1)
b = lib._device(fn, x0, x1, flags=_lib.FLAG_FORCE_EXACT)
torch.cuda.synchronize()
u = np.uint64 if width == 64 else np.uint32
A0, A1, B0, B1 = (t.cpu().numpy() for t in (a.value, a.error, b.value, b.error))
bad = np.nonzero((A0.view(u) != B0.view(u)) | (A1.view(u) != B1.view(u)))[0]
for i in bad[:10]:
    print(i, float(g["x0"][i]).hex(), float(g["x1"][i]).hex(), "fast", float(A0[i]).hex(),
          float(A1[i]).hex(), "exact", float(B0[i]).hex(), float(B1[i]).hex())
print(len(bad), "mismatches")
