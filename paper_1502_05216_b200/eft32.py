"""Binary32 lane of the element-wise EFTs and twofold arithmetic (reference
pkg/src/twofold/eft32.py:36-214): the same names and contracts as eft.py,
every operand and result an exact binary32 value, evaluated by the binary32
kernels of csrc/tf_eft.cu (native IEEE binary32 ops == the reference's
r32-narrowed double ops)."""

from __future__ import annotations

from ._eftops import LANES, Arith
from .eft import SplitPair, Twofold, get_default_backend

__all__ = ["fast_two_sum", "two_sum", "two_diff", "split", "two_prod_fma", "two_prod_dv",
           "fma_sim", "renorm_fast", "renorm", "arith", "t_add", "t_add_d", "Arith",
           "Twofold", "SplitPair"]

_L = LANES[32]

fast_two_sum = _L.fast_two_sum
two_sum = _L.two_sum
two_diff = _L.two_diff
split = _L.split
two_prod_fma = _L.two_prod_fma
two_prod_dv = _L.two_prod_dv
fma_sim = _L.fma_sim
renorm_fast = _L.renorm_fast
renorm = _L.renorm
t_add = _L.t_add
t_add_d = _L.t_add_d


def arith(backend: str | None = None) -> Arith:
    return _L.arith(get_default_backend() if backend is None else backend)
