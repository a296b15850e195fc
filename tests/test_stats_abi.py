"""tf_reduce_stats (include/twofold_b200.h): the C ABI's
order-independent merge of shard statistics -- counts and sums add, maxima
max (reference audit.py:205-269; SPEC.md "merge of (sum, max, count) is
order-independent").  Host code only: runs without a GPU."""

import ctypes
import math
import random

import pytest

from paper_1502_05216_b200 import _lib
from paper_1502_05216_b200.dist import to_record


def _rand_record(rng):
    r = _lib.TfStats()
    for k in _lib.STATS_COUNT_KEYS:
        setattr(r, k, rng.randrange(0, 1 << 40))
    r.err_sum = rng.random() * 1e-20
    r.err_max = rng.choice([rng.random() * -100.0, float("-inf"), float("nan")])
    return r


def test_merge_is_sum_and_max_in_any_order():
    rng = random.Random(5)
    parts = [_rand_record(rng) for _ in range(9)]
    whole = _lib.reduce_stats_c(parts)
    for k in _lib.STATS_COUNT_KEYS:
        assert getattr(whole, k) == sum(getattr(p, k) for p in parts)
    assert math.isclose(whole.err_sum, sum(p.err_sum for p in parts), rel_tol=1e-12)
    finite = [p.err_max for p in parts if not math.isnan(p.err_max)]
    assert whole.err_max == max(finite)
    rng.shuffle(parts)
    again = _lib.reduce_stats_c(parts)
    assert bytes(again)[:64] == bytes(whole)[:64]      # counts: exactly order-independent
    assert again.err_max == whole.err_max
    # merging merged halves gives the same record (associativity of the merge)
    h = _lib.reduce_stats_c([_lib.reduce_stats_c(parts[:4]), _lib.reduce_stats_c(parts[4:])])
    assert bytes(h)[:64] == bytes(whole)[:64] and h.err_max == whole.err_max


def test_empty_and_argument_errors():
    L = _lib.load()
    out = _lib.TfStats()
    assert L.tf_reduce_stats(None, 0, ctypes.byref(out)) == _lib.TF_OK
    assert out.n == 0 and out.err_max == float("-inf")
    assert L.tf_reduce_stats(None, 3, ctypes.byref(out)) == _lib.TF_ERR_ARG
    assert L.tf_reduce_stats(None, 0, None) == _lib.TF_ERR_ARG
    with pytest.raises(ValueError):
        _lib.check(L.tf_reduce_stats(None, -1, ctypes.byref(out)), "tf_reduce_stats")


def test_record_layout_matches_header():
    assert ctypes.sizeof(_lib.TfStats) == 80
    r = to_record({"n": 5, "z0_mismatch": 1, "z1_bit_mismatch": 2, "worst_rel_log2": -101.5})
    assert (r.n, r.z0_mismatch, r.z1_mismatch, r.err_max) == (5, 1, 2, -101.5)
