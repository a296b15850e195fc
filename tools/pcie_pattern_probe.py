"""Which part of the host pipeline costs time?  Copy patterns over 2 x 2^24
binary64 arrays in and out (the e2e step of one function), without kernels:
  bulk      one H2D stream and one D2H stream, whole arrays, no dependencies
  ring-c    the tf_eval_host copy pattern (chunk c, 4-slot ring, H2D -> D2H
            dependency per chunk through events), kernel replaced by nothing
  ring-c+k  the same with the kernel between (tf_eval on the compute stream)
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib  # noqa: E402

n = 1 << 24
x0 = torch.empty(n, dtype=torch.float64).uniform_(-1, 1)
hs = [x0.pin_memory(), (x0 * 2.0 ** -60).pin_memory()]     # in-band twofolds
ho = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
dev_in = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
dev_out = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(2)]
s_in, s_comp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
L = _lib.ensure_device(0)


def timed(name, fn, reps=5, sync_each=False):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
        if sync_each:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"{name:24s} {dt * 1e3:7.2f} ms  {4 * n * 8 / dt / 1e9:6.1f} GB/s both ways", flush=True)


def bulk():
    with torch.cuda.stream(s_in):
        for a in range(2):
            dev_in[a].copy_(hs[a], non_blocking=True)
    with torch.cuda.stream(s_out):
        for a in range(2):
            ho[a].copy_(dev_out[a], non_blocking=True)


def ring(c, kernel, ring_n=4, kev=None):
    def run():
        free = [None] * ring_n
        for k, off in enumerate(range(0, n, c)):
            m = min(c, n - off)
            sl = k % ring_n
            if free[sl] is not None:
                s_in.wait_event(free[sl])
            with torch.cuda.stream(s_in):
                for a in range(2):
                    dev_in[a][sl * c:sl * c + m].copy_(hs[a][off:off + m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_in)
            s_comp.wait_event(ev)
            if kernel == "d2d":
                with torch.cuda.stream(s_comp):
                    for a in range(2):
                        dev_out[a][sl * c:sl * c + m].copy_(dev_in[a][sl * c:sl * c + m])
            elif kernel:
                if kev is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(s_comp)
                rc = L.tf_eval(_lib.FN_CODES["texpm1"], 64, dev_in[0][sl * c:].data_ptr(),
                               dev_in[1][sl * c:].data_ptr(), dev_out[0][sl * c:].data_ptr(),
                               dev_out[1][sl * c:].data_ptr(), m, s_comp.cuda_stream, 0)
                assert rc == 0
                if kev is not None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(s_comp)
                    kev.append((e0, e1))
            ev2 = torch.cuda.Event()
            ev2.record(s_comp)
            s_out.wait_event(ev2)
            with torch.cuda.stream(s_out):
                for a in range(2):
                    ho[a][off:off + m].copy_(dev_out[a][sl * c:sl * c + m], non_blocking=True)
                ev3 = torch.cuda.Event()
                ev3.record(s_out)
            free[sl] = ev3
    return run


timed("bulk (upper bound)", bulk)


def host_api(c):
    def run():
        rc = L.tf_eval_host(_lib.FN_CODES["texpm1"], 64, hs[0].data_ptr(), hs[1].data_ptr(),
                            ho[0].data_ptr(), ho[1].data_ptr(), n, c, None, 0)
        assert rc == 0
    return run


for c in (1 << 20, 1 << 21, 1 << 22):
    timed(f"tf_eval_host 2^{c.bit_length() - 1}", host_api(c))
if os.environ.get("HOST_ONLY"):
    sys.exit(0)
for c in (1 << 20, 1 << 21, 1 << 22):
    timed(f"ring 2^{c.bit_length() - 1} copies only", ring(c, False))
    timed(f"ring 2^{c.bit_length() - 1} + kernel", ring(c, True))
timed("ring 2^21 copies, ring 8", ring(1 << 21, False, 8))
timed("ring 2^21 + d2d copy kernel", ring(1 << 21, "d2d"))
# per-call latency: a host synchronisation after every repetition (the API returns host results)
timed("bulk, sync each", bulk, sync_each=True)
for c in (1 << 19, 1 << 20, 1 << 21):
    timed(f"ring 2^{c.bit_length() - 1} copies, sync each", ring(c, False), sync_each=True)
    timed(f"ring 2^{c.bit_length() - 1} + kernel, sync each", ring(c, True), sync_each=True)
kev = []
f = ring(1 << 21, True, kev=kev)
f()
torch.cuda.synchronize()
print("kernel ms inside the pipeline:", [round(a.elapsed_time(b), 3) for a, b in kev])
kev.clear()
s_comp.synchronize()
for _ in range(3):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s_comp)
    L.tf_eval(_lib.FN_CODES["texpm1"], 64, dev_in[0].data_ptr(), dev_in[1].data_ptr(),
              dev_out[0].data_ptr(), dev_out[1].data_ptr(), 1 << 21, s_comp.cuda_stream, 0)
    e1.record(s_comp)
    torch.cuda.synchronize()
    print("kernel ms alone:", round(e0.elapsed_time(e1), 3))
