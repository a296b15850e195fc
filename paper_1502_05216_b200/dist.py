"""Multi-GPU plumbing for the sharded hot path.

The twofold functions are elementwise, so G GPUs take contiguous shards of the
global index range and never exchange data while evaluating; the only
collective is one tiny reduction of error statistics afterwards (and the
max-over-ranks timing reduction of the benchmark).  Everything here works with
any torch.distributed backend: NCCL over NVLink on the B200 box, gloo in the
CPU tests (tests/test_multi_gloo.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

# counters summed across ranks / maxima taken across ranks
SUM_KEYS = ("n", "z0_mismatch", "z0_gt1ulp", "tol_violations", "class_mismatch")
MAX_KEYS = ("worst_rel_log2",)


def shard_range(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [start, start+count) of rank in a world of size `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    lo = n_global * rank // world
    hi = n_global * (rank + 1) // world
    return lo, hi - lo


def _active() -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def reduce_stats(stats: dict, device=None) -> dict:
    """Sum the counters and max the maxima of a per-rank stats dict (one
    all-reduce each, a few dozen bytes)."""
    out = dict(stats)
    if not _active():
        return out
    dev = device if device is not None else torch.device("cpu")
    s = torch.tensor([float(stats.get(k, 0)) for k in SUM_KEYS], dtype=torch.float64, device=dev)
    m = torch.tensor([float(stats.get(k, float("-inf"))) for k in MAX_KEYS], dtype=torch.float64,
                     device=dev)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    for k, v in zip(SUM_KEYS, s.tolist()):
        out[k] = int(v)
    for k, v in zip(MAX_KEYS, m.tolist()):
        out[k] = v
    return out


def max_over_ranks(value: float, device=None) -> float:
    if not _active():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device or torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    if _active():
        dist.barrier()
