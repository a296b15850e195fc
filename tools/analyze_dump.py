import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from oracle.compare import compare, same_bits, ulp_distance
from paper_1502_05216_b200 import workloads
d = np.load('gpurun_out/dump.npz')
N = int(os.environ.get("DUMP_N", 1 << 18))
show = int(os.environ.get("SHOW", 6))
def h(x): return float(x).hex()
for k in d.files:
    a0, a1, b0, b1 = d[k]
    if k.startswith('g_'):
        _, fn, w = k.split('_'); w = int(w)
        g = np.load(f'tests/golden/golden_{fn}_f{w}.npz'); x0, x1, r0, r1 = g['x0'], g['x1'], g['z0'], g['z1']
    else:
        cfg = k[2:]; fn, w, dist, _ = workloads.CONFIGS[cfg]
        x0, x1 = workloads.generate(dist, 0, N, seed=1)
        r0, r1 = O.evaluate(fn, w, x0, x1, backend='dv')
    r = compare(a0, a1, r0, r1, w); fe = compare(a0, a1, b0, b1, w)
    print(f"== {k}: z0mis={r['z0_mismatch']} hist={r['z0_ulp_hist']} tolv={r['tol_violations']} tolv|z0={r['tol_violations_given_z0_match']} cls={r['class_mismatch']} | fast-vs-exact z0={fe['z0_mismatch']} z1={fe['z1_bit_mismatch']}")
    bad = r['bad_idx'][:show]
    for i in bad:
        print(f"   BAD x=({h(x0[i])},{h(x1[i])}) gpu=({h(a0[i])},{h(a1[i])}) exact=({h(b0[i])},{h(b1[i])}) ref=({h(r0[i])},{h(r1[i])})")
    ud = ulp_distance(a0, r0)
    big = np.nonzero((~same_bits(a0, r0)) & ((ud > 1) | (ud < 0)))[0][:show]
    for i in big:
        print(f"   ULP>1 x=({h(x0[i])},{h(x1[i])}) gpu=({h(a0[i])},{h(a1[i])}) exact=({h(b0[i])},{h(b1[i])}) ref=({h(r0[i])},{h(r1[i])})")
    fx = np.nonzero(~(same_bits(a0, b0) & same_bits(a1, b1)))[0][:show]
    for i in fx:
        print(f"   FAST!=EXACT x=({h(x0[i])},{h(x1[i])}) gpu=({h(a0[i])},{h(a1[i])}) exact=({h(b0[i])},{h(b1[i])}) ref=({h(r0[i])},{h(r1[i])})")
