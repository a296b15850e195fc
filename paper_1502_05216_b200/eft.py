"""Twofold value type, backend selection and the binary64 EFT / twofold
arithmetic ops (reference pkg/src/twofold/eft.py:51-317).

``Twofold(value, error)`` is the same NamedTuple as the reference's; its fields
may hold Python floats, numpy arrays or torch tensors.  The "fma"/"dv"
backend names select the exact-product residual of the element-wise ops
(csrc/tf_eft.cu: one hardware FMA, or the Dekker-Veltkamp split sequence, bit
for bit the reference's); the exp/log kernels always use the FMA.

The ops take scalars, numpy arrays or torch tensors (CUDA tensors stay on
their device) and run on the GPU; eft32.py is the binary32 lane.
"""

from __future__ import annotations

import os
from typing import Any, NamedTuple

__all__ = ["Twofold", "SplitPair", "set_default_backend", "get_default_backend",
           "fast_two_sum", "two_sum", "two_diff", "split", "two_prod_fma", "two_prod_dv",
           "fma_sim", "renorm_fast", "renorm", "Arith", "arith", "t_add", "t_add_d", "t_mul",
           "t_mul_d", "t_div", "t_sqrt"]


class Twofold(NamedTuple):
    """Unevaluated sum value + error; error may have any magnitude."""

    value: Any
    error: Any


class SplitPair(NamedTuple):
    """Exact split x == hi + lo (kept for API compatibility)."""

    hi: Any
    lo: Any


def _initial_backend() -> str:
    env = os.environ.get("TWOFOLD_BACKEND", "").strip().lower()
    return env if env in ("fma", "dv") else "fma"


_default_backend = _initial_backend()


def set_default_backend(backend: str) -> None:
    global _default_backend
    if backend not in ("fma", "dv"):
        raise ValueError(f"unknown backend {backend!r}; expected 'fma' or 'dv'")
    _default_backend = backend


def get_default_backend() -> str:
    return _default_backend


# ---- element-wise EFTs / twofold arithmetic, binary64 lane (eft.py:77-237)
def _lane():
    from ._eftops import LANES

    return LANES[64]


def fast_two_sum(a, b):
    """Exact a + b as value + error; requires |a| >= |b| or a == 0."""
    return _lane().fast_two_sum(a, b)


def two_sum(a, b):
    """Exact a + b as value + error, no magnitude precondition."""
    return _lane().two_sum(a, b)


def two_diff(a, b):
    """Exact a - b as value + error (the corrected six-step sequence)."""
    return _lane().two_diff(a, b)


def split(x):
    """Dekker split x == hi + lo, each part at most 26/27 bits."""
    return _lane().split(x)


def two_prod_fma(x, y):
    return _lane().two_prod_fma(x, y)


def two_prod_dv(x, y):
    return _lane().two_prod_dv(x, y)


def fma_sim(x, y, z):
    return _lane().fma_sim(x, y, z)


def renorm_fast(x):
    return _lane().renorm_fast(x)


def renorm(x):
    return _lane().renorm(x)


def arith(backend: str | None = None):
    """Arithmetic bundle for the given backend ("fma" or "dv")."""
    return _lane().arith(_default_backend if backend is None else backend)


def t_add(x, y):
    return _lane().t_add(x, y)


def t_add_d(x, b):
    return _lane().t_add_d(x, b)


def t_mul(x, y):
    return _lane().t_mul(x, y, _default_backend)


def t_mul_d(x, b):
    return _lane().t_mul_d(x, b, _default_backend)


def t_div(x, y):
    return _lane().t_div(x, y, _default_backend)


def t_sqrt(x):
    return _lane().t_sqrt(x, _default_backend)


def __getattr__(name):
    if name == "Arith":
        from ._eftops import Arith

        return Arith
    raise AttributeError(name)
