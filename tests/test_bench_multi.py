"""bench.py's own multi-rank machinery on CPU:

* `--gpus 2` outside torchrun relaunches itself under torch.distributed.run
  with two ranks; the reference arm (CPU port, rank 0 only) then prints ONE
  line with n_gpus = 2 and the same config the GPU arm prints;
* bench's slice assignment and its parity merge (the run's one small
  collective: tf_reduce_stats over an all-gather) reproduce the
  single-process statistics over the whole range, over gloo with 2 ranks.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

N = 5000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_gpus2_relaunches_reference_arm():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
           "--steps", "1", "--warmup", "3", "--ref-sample", "4096", "--py-ref-sample", "0"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    sys.path.insert(0, ROOT)
    import bench

    assert rec["impl"] == "reference" and rec["n_gpus"] == 2
    assert rec["config"] == bench.config_for(2)
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["value"] > 0
    assert rec["cpu_baseline"]["kind"] == "port"


@pytest.mark.gpu
def test_bench_gpu_arm_two_ranks_code_path():
    """The GPU arm's N > 1 path -- relaunch, contiguous shards, max-over-ranks
    timing, the parity merge -- with two ranks over gloo.  On a one-GPU box both
    ranks share the device (independent kernels, nothing waits across ranks),
    so this checks the code path, not the scaling."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
           "--steps", "3", "--warmup", "3", "--headline-only", "--no-e2e", "--no-cpu",
           "--parity-sample", "65536", "--parity-host", "4096"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["value"] > 0
    assert rec["config"]["elements_per_function_per_gpu"] == (1 << 29)
    for fn in ("texp", "tlog"):
        n, z0mm, gt1, tol, tolz, cls = rec["parity_cfg5"][fn][:6]
        # the parity sample is split over the ranks: the merged count is the sample
        assert n == 65536 and gt1 == 0 and tol == 0 and tolz == 0 and cls == 0


def test_bench_world_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from oracle import oracle as O
        from oracle.compare import compare
        from paper_1502_05216_b200 import workloads

        start, n = bench.shard(N, rank, world)
        x0, x1 = workloads.generate("logu64s", start, n, seed=bench.SEED)
        z = O.evaluate("tlog", 64, x0, x1, backend="fma", nthreads=1)
        r = O.evaluate("tlog", 64, x0, x1, backend="dv", nthreads=1, libm64="glibc")
        merged = bench._reduce(compare(*z, *r, 64), None)
        q.put((rank, start, n, bench._compact(merged)))
    finally:
        dist.destroy_process_group()


def test_bench_shards_and_parity_merge_two_ranks():
    from oracle import oracle as O
    from oracle.compare import compare
    from paper_1502_05216_b200 import workloads

    sys.path.insert(0, ROOT)
    import bench

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == 0 and res[0][2] + res[1][2] == N and res[1][1] == res[0][2]
    x0, x1 = workloads.generate("logu64s", 0, N, seed=bench.SEED)
    whole = bench._compact(compare(*O.evaluate("tlog", 64, x0, x1, backend="fma"),
                                   *O.evaluate("tlog", 64, x0, x1, backend="dv"), 64))
    for _, _, _, got in res:
        assert got[:6] == whole[:6]
        assert np.isclose(got[6], whole[6])
