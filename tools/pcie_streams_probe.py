import time, torch
n = 1 << 26
H = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
D = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4)]
S = [torch.cuda.Stream() for _ in range(4)]
def run(pairs):
    for k, (dirn, i) in enumerate(pairs):
        with torch.cuda.stream(S[k]):
            if dirn == "h2d": D[i].copy_(H[i], non_blocking=True)
            else: H[i].copy_(D[i], non_blocking=True)
def bw(name, pairs, reps=5):
    run(pairs); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): run(pairs)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"{name:30s} {len(pairs) * n * 8 / dt / 1e9:7.1f} GB/s", flush=True)
bw("h2d x1", [("h2d", 0)])
bw("h2d x2 streams", [("h2d", 0), ("h2d", 1)])
bw("d2h x1", [("d2h", 0)])
bw("d2h x2 streams", [("d2h", 0), ("d2h", 1)])
bw("h2d+d2h 1+1", [("h2d", 0), ("d2h", 1)])
bw("h2d+d2h 2+2", [("h2d", 0), ("h2d", 1), ("d2h", 2), ("d2h", 3)])
