"""Twofold value type and backend selection (reference pkg/src/twofold/eft.py:51-62,
280-301).

``Twofold(value, error)`` is the same NamedTuple as the reference's; its fields
may hold Python floats, numpy arrays or torch tensors.  The "fma"/"dv"
backend names are accepted for signature compatibility: the B200 kernels
always form the exact product residual with one hardware FMA.
"""

from __future__ import annotations

import os
from typing import Any, NamedTuple

__all__ = ["Twofold", "SplitPair", "set_default_backend", "get_default_backend"]


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
