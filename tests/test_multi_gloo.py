"""Multi-rank path on CPU (gloo, world_size 2): contiguous shards of the global
index range, per-rank evaluation, and the single small all-reduce of error
statistics (paper_1502_05216_b200.dist) must reproduce the single-process
result over the whole range.  The GPU run uses the same code over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

N = 6000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from oracle.compare import compare
        from paper_1502_05216_b200 import dist as D
        from paper_1502_05216_b200 import workloads

        start, count = D.shard_range(N, rank, world)
        x0, x1 = workloads.generate("exp64s", start, count, seed=9)
        z = O.evaluate("texp", 64, x0, x1, backend="fma", nthreads=1)
        r = O.evaluate("texp", 64, x0, x1, backend="dv", nthreads=1)
        local = compare(*z, *r, 64)
        total = D.reduce_stats(local)
        t = D.max_over_ranks(float(rank + 1))
        D.barrier()
        q.put((rank, start, count, total, t))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover():
    from paper_1502_05216_b200.dist import shard_range

    for world in (1, 2, 3, 8):
        spans = [shard_range(1001, r, world) for r in range(world)]
        assert spans[0][0] == 0
        for (a, n), (b, _) in zip(spans, spans[1:]):
            assert a + n == b
        assert spans[-1][0] + spans[-1][1] == 1001
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_two_rank_gloo_stats_reduce():
    from oracle import oracle as O
    from oracle.compare import compare
    from paper_1502_05216_b200 import workloads

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x0, x1 = workloads.generate("exp64s", 0, N, seed=9)
    whole = compare(*O.evaluate("texp", 64, x0, x1, backend="fma"),
                    *O.evaluate("texp", 64, x0, x1, backend="dv"), 64)
    for rank, start, count, total, tmax in res:
        assert tmax == 2.0
        for k in ("n", "z0_mismatch", "z0_gt1ulp", "tol_violations", "class_mismatch"):
            assert total[k] == whole[k], k
        assert np.isclose(total["worst_rel_log2"], whole["worst_rel_log2"])
    assert res[0][1] == 0 and res[1][1] == res[0][2]
