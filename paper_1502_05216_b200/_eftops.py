"""Array EFT / twofold-arithmetic ops on the B200 (the kernels of
csrc/tf_eft.cu through tf_eft).  Shared by eft.py (binary64 lane) and
eft32.py (binary32 lane); see those modules for the public names.

Operands may be Python floats, numpy arrays, or torch tensors (CPU or CUDA);
CUDA tensors are evaluated in place on their device and stream, everything
else is copied to the current CUDA device and the result copied back (the
arithmetic always runs in the kernels -- there is no CPU fallback).
"""

from __future__ import annotations

from typing import Callable, NamedTuple

import numpy as np

from . import _lib


class Arith(NamedTuple):
    """Twofold arithmetic bound to one exact-residual backend (eft.py:240-251)."""

    backend: str
    t_add: Callable
    t_add_d: Callable
    t_mul: Callable
    t_mul_d: Callable
    t_div: Callable
    t_sqrt: Callable
    prod_err: Callable
    rem: Callable


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


class Lane:
    """The ops of one float width."""

    def __init__(self, width: int):
        self.width = width
        self.np = np.float64 if width == 64 else np.float32

    # ---- operand plumbing
    def _prep(self, args):
        import torch

        dt = torch.float64 if self.width == 64 else torch.float32
        cuda = next((a for a in args if _is_torch(a) and a.is_cuda), None)
        scalar = all(not _is_torch(a) and np.ndim(a) == 0 for a in args)
        if cuda is not None:
            dev = cuda.device
        else:
            if not torch.cuda.is_available():
                raise RuntimeError("no CUDA device visible: the twofold kernels need a B200 "
                                   "(sm_100a); there is no CPU fallback")
            dev = torch.device("cuda", torch.cuda.current_device())
        ts = []
        for a in args:
            if _is_torch(a):
                t = a.to(device=dev, dtype=dt)
            else:
                t = torch.as_tensor(np.asarray(a, dtype=self.np), device=dev)
            ts.append(t)
        shape = torch.broadcast_shapes(*(t.shape for t in ts))
        ts = [t.expand(shape).contiguous() for t in ts]
        return ts, dev, ("scalar" if scalar else "cuda" if cuda is not None else "host")

    def _finish(self, z0, z1, kind, tf):
        if kind == "cuda":
            return tf(z0, z1)
        a0, a1 = z0.cpu().numpy(), z1.cpu().numpy()
        if kind == "scalar":
            return tf(float(a0.reshape(-1)[0]), float(a1.reshape(-1)[0]))
        return tf(a0, a1)

    def run(self, op: str, a0, a1=None, b0=None, b1=None, backend: str = "fma", tf=None):
        import torch

        from .eft import SplitPair, Twofold

        if backend not in ("fma", "dv"):
            raise ValueError(f"unknown backend {backend!r}; expected 'fma' or 'dv'")
        tf = tf or (SplitPair if op == "split" else Twofold)
        present = [a for a in (a0, a1, b0, b1) if a is not None]
        ts, dev, kind = self._prep(present)
        it = iter(ts)
        x0 = next(it)
        x1 = next(it) if a1 is not None else None
        y0 = next(it) if b0 is not None else None
        y1 = next(it) if b1 is not None else None
        z0 = torch.empty_like(x0)
        z1 = torch.empty_like(x0)
        n = x0.numel()
        L = _lib.ensure_device(dev.index)
        ptr = (lambda t: t.data_ptr() if t is not None else None)
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            _lib.check(L.tf_eft(_lib.OP_CODES[op], self.width, 1 if backend == "dv" else 0,
                                ptr(x0), ptr(x1), ptr(y0), ptr(y1), z0.data_ptr(),
                                z1.data_ptr(), n, stream), f"tf_eft({op})")
        if kind != "cuda":
            torch.cuda.synchronize(dev)
        return self._finish(z0, z1, kind, tf)

    # ---- the reference's free functions (eft.py:77-171)
    def fast_two_sum(self, a, b):
        return self.run("fast_two_sum", a, b0=b)

    def two_sum(self, a, b):
        return self.run("two_sum", a, b0=b)

    def two_diff(self, a, b):
        return self.run("two_diff", a, b0=b)

    def split(self, x):
        return self.run("split", x)

    def two_prod_fma(self, x, y):
        return self.run("two_prod", x, b0=y, backend="fma")

    def two_prod_dv(self, x, y):
        return self.run("two_prod", x, b0=y, backend="dv")

    def fma_sim(self, x, y, z):
        """(z + p) + t with (p, t) = two_prod_dv(x, y) (eft.py:152-160)."""
        p = self.two_prod_dv(x, y)
        s = self.t_add_d(p, z, backend="dv")
        return self.renorm_fast(s).value

    def renorm_fast(self, x):
        return self.run("renorm_fast", x[0], x[1])

    def renorm(self, x):
        return self.run("renorm", x[0], x[1])

    def t_add(self, x, y, backend="fma"):
        return self.run("t_add", x[0], x[1], y[0], y[1])

    def t_add_d(self, x, b, backend="fma"):
        return self.run("t_add_d", x[0], x[1], b)

    def t_mul(self, x, y, backend="fma"):
        return self.run("t_mul", x[0], x[1], y[0], y[1], backend=backend)

    def t_mul_d(self, x, b, backend="fma"):
        return self.run("t_mul_d", x[0], x[1], b, backend=backend)

    def t_div(self, x, y, backend="fma"):
        return self.run("t_div", x[0], x[1], y[0], y[1], backend=backend)

    def t_sqrt(self, x, backend="fma"):
        return self.run("t_sqrt", x[0], x[1], backend=backend)

    def arith(self, backend: str) -> Arith:
        """Arithmetic bundle for one backend (eft.py:202-251, 275-283)."""
        if backend not in ("fma", "dv"):
            raise ValueError(f"unknown backend {backend!r}; expected 'fma' or 'dv'")

        def prod_err(x, y, v):
            # the exact residual x*y - v for v = fl(x*y)
            return self.run("two_prod", x, b0=y, backend=backend).error

        def rem(q, b, a):
            # a - q*b for the exact-remainder case (division / sqrt, eft.py:267-272):
            # (a + p) + t with (p, t) = -two_prod(q, b), p + a exact by Sterbenz
            v, e = self.run("two_prod", q, b0=b, backend=backend)
            return self.renorm_fast(self.t_add_d((-v, -e), a)).value

        return Arith(
            backend,
            lambda x, y: self.t_add(x, y),
            lambda x, b: self.t_add_d(x, b),
            lambda x, y: self.t_mul(x, y, backend),
            lambda x, b: self.t_mul_d(x, b, backend),
            lambda x, y: self.t_div(x, y, backend),
            lambda x: self.t_sqrt(x, backend),
            prod_err,
            rem,
        )


LANES = {64: Lane(64), 32: Lane(32)}
