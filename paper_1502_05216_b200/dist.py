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

# stats-dict keys carried by the C record struct tf_stats (include/twofold_b200.h);
# worst_rel_log2 travels in err_max
RECORD_KEYS = {"n": "n", "z0_mismatch": "z0_mismatch", "z0_gt1ulp": "z0_gt1ulp",
               "tol_violations": "tol_violations", "class_mismatch": "class_mismatch",
               "z1_bit_mismatch": "z1_mismatch", "included": "included", "warnings": "warnings",
               "err_sum": "err_sum", "worst_rel_log2": "err_max"}


def shard_range(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [start, start+count) of rank in a world of size `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    lo = n_global * rank // world
    hi = n_global * (rank + 1) // world
    return lo, hi - lo


def _active() -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def to_record(stats: dict):
    """Pack a stats dict (oracle.compare / audit counters) into a tf_stats record."""
    from ._lib import TfStats

    r = TfStats()
    r.err_max = float("-inf")
    for k, f in RECORD_KEYS.items():
        if k in stats and stats[k] is not None:
            setattr(r, f, type(getattr(r, f))(stats[k]))
    return r


def reduce_stats(stats: dict, device=None) -> dict:
    """Merge a per-rank stats dict over all ranks: each rank contributes its
    fixed-size tf_stats record (80 bytes) to one all-gather, and the records
    merge with the C ABI's tf_reduce_stats (counts and sums add, maxima max).
    Integer counters outside the record (e.g. *_given_z0_match) are summed
    with one all-reduce; list-valued entries (diagnostic indices, histograms)
    stay per-rank."""
    out = dict(stats)
    if not _active():
        return out
    from ._lib import TfStats, reduce_stats_c

    dev = device if device is not None else torch.device("cpu")
    world = dist.get_world_size()
    rec = bytes(to_record(stats))
    mine = torch.frombuffer(bytearray(rec), dtype=torch.uint8).to(dev)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    merged = reduce_stats_c([TfStats.from_buffer_copy(bytes(p.cpu().numpy())) for p in parts])
    for k, f in RECORD_KEYS.items():
        if k in stats:
            v = getattr(merged, f)
            out[k] = v if isinstance(v, float) else int(v)
    extra = sorted(k for k, v in stats.items()
                   if k not in RECORD_KEYS and isinstance(v, int) and not isinstance(v, bool))
    if extra:
        t = torch.tensor([float(stats[k]) for k in extra], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        for k, v in zip(extra, t.tolist()):
            out[k] = int(v)
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
