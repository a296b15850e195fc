"""Drop-in twofold exp/log surface, B200 edition.

Mirrors the reference public API (pkg/src/twofold/explog.py:44-62, 69-349;
__init__.py:19-57): ``api(width, backend=None) -> ExpLog``, ``ExpLog.texp /
texpm1 / tlog / tlog1p``, ``ExpLog.function(name)``, ``get_function(name,
width, backend=None)``, ``FAMILIES``, ``FUNCTION_NAMES``, ``DOTTED_ARG``,
``COUPLED_ARG``, ``TWOFOLD_ARG``, ``family_of``.  Same names, argument meaning
and error behaviour (ValueError for a bad width, backend or function name).

What changes is the operand: besides the reference's scalar pair ``(x0, x1)``
an argument may be a pair of arrays -- CUDA tensors (evaluated on their device
and the current stream, results allocated there), CPU tensors or numpy arrays
(copied through pinned staging buffers, results returned on the host).  Every
evaluation runs the hand-written sm_100a kernels of libtwofold_b200.so; there
is no CPU fallback.

All twenty reference functions are served by the same admission-band kernels
(tf_fast.cuh fast_eval): ``texpp``/``texpm1p`` are ``texp``/``texpm1``, the
p-functions return renorm_fast of the cores, the dotted t-functions run their
twofold twins with x1 = 0, and the coupled-argument log functions skip the
renormalisation (explog.py:101-325).
DOTTED_ARG functions take a plain argument (a scalar, array or tensor, not a
pair).  COUPLED_ARG functions assume |x1| <= ulp(x0)/2 like the reference;
where the reference raises OverflowError for a non-coupled argument
(math.ldexp, explog.py:192) the GPU returns a value instead of raising.
"""

from __future__ import annotations

import ctypes
from ctypes import byref
from functools import lru_cache

import numpy as np

from . import _lib
from .eft import Twofold, get_default_backend
from .params import params_for_width

__all__ = ["ExpLog", "api", "get_function", "FAMILIES", "FUNCTION_NAMES", "DOTTED_ARG",
           "COUPLED_ARG", "TWOFOLD_ARG", "family_of"]

FAMILIES = {
    "exp": ("pexp0", "texp0", "texp", "texpp", "pexp"),
    "expm1": ("pexpm10", "texpm10", "texpm1", "texpm1p", "pexpm1"),
    "log": ("plog0", "tlog0", "tlogp", "tlog", "plog"),
    "log1p": ("plog1p0", "tlog1p0", "tlog1pp", "tlog1p", "plog1p"),
}
FUNCTION_NAMES = tuple(name for fam in FAMILIES.values() for name in fam)
DOTTED_ARG = frozenset(n for n in FUNCTION_NAMES if n.endswith("0"))
COUPLED_ARG = frozenset(("texpp", "pexp", "texpm1p", "pexpm1", "tlogp", "plog", "tlog1pp",
                         "plog1p"))
TWOFOLD_ARG = frozenset(("texp", "texpm1", "tlog", "tlog1p"))

HOST_CHUNK = 1 << 20  # tf_eval_host's default chunk (elements per pipelined transfer)


def family_of(name: str) -> str:
    for fam, names in FAMILIES.items():
        if name in names:
            return fam
    raise ValueError(f"unknown function {name!r}")


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _span(t):
    lo = t.data_ptr()
    return lo, lo + t.numel() * t.element_size()


def _overlaps(a, b) -> bool:
    if a.numel() == 0 or b.numel() == 0:
        return False
    (a0, a1), (b0, b1) = _span(a), _span(b)
    return a0 < b1 and b0 < a1


def _same_span(a, b) -> bool:
    return _span(a) == _span(b)


class ExpLog:
    """Twofold exponent and logarithm functions for one float width."""

    def __init__(self, width: int, backend: str | None = None):
        params = params_for_width(width)
        if backend is None:
            backend = get_default_backend()
        if backend not in ("fma", "dv"):
            raise ValueError(f"unknown backend {backend!r}; expected 'fma' or 'dv'")
        self.width = width
        # Both reference backends name an exact-product residual; the GPU computes
        # it with one hardware FMA (bitwise equal to "dv" except subnormal z1).
        self.backend = backend
        self.params = params
        self._np = np.float64 if width == 64 else np.float32
        self._ct = ctypes.c_double if width == 64 else ctypes.c_float

    # ---- the four twofold-argument functions (explog.py:115, 149, 244, 314)
    def texp(self, x, out=None):
        """Twofold e**(x0+x1); value part = correctly rounded exp(x0)."""
        return self._call("texp", x, out)

    def texpm1(self, x, out=None):
        """Twofold e**(x0+x1) - 1; value part = correctly rounded expm1(x0)."""
        return self._call("texpm1", x, out)

    def tlog(self, y, out=None):
        """Twofold ln of any twofold; value part = correctly rounded log(y0)."""
        return self._call("tlog", y, out)

    def tlog1p(self, y, out=None):
        """Twofold ln(1 + y0 + y1); value part = correctly rounded log1p(y0)."""
        return self._call("tlog1p", y, out)

    # ---- the sixteen siblings (explog.py:101-325)
    def pexp0(self, x, out=None):
        """Pair e**x of a plain x (pexp0, explog.py:101-103)."""
        return self._call("pexp0", x, out)

    def texp0(self, x, out=None):
        """Twofold e**x of a plain x (texp0, explog.py:105-113)."""
        return self._call("texp0", x, out)

    def texpp(self, x, out=None):
        """Twofold e**(x0+x1) of a coupled twofold (texpp, explog.py:127-129)."""
        return self._call("texpp", x, out)

    def pexp(self, x, out=None):
        """Renormalised pair e**(x0+x1) of a coupled twofold (pexp, explog.py:131-133)."""
        return self._call("pexp", x, out)

    def pexpm10(self, x, out=None):
        """Pair e**x - 1 of a plain x (pexpm10, explog.py:135-137)."""
        return self._call("pexpm10", x, out)

    def texpm10(self, x, out=None):
        """Twofold e**x - 1 of a plain x (texpm10, explog.py:139-147)."""
        return self._call("texpm10", x, out)

    def texpm1p(self, x, out=None):
        """Twofold e**(x0+x1) - 1 of a coupled twofold (texpm1p, explog.py:162-163)."""
        return self._call("texpm1p", x, out)

    def pexpm1(self, x, out=None):
        """Renormalised pair e**(x0+x1) - 1 (pexpm1, explog.py:165-166)."""
        return self._call("pexpm1", x, out)

    def plog0(self, y, out=None):
        """Pair ln y of a plain y (plog0, explog.py:225-232)."""
        return self._call("plog0", y, out)

    def tlog0(self, y, out=None):
        """Twofold ln y of a plain y (tlog0, explog.py:234-237)."""
        return self._call("tlog0", y, out)

    def tlogp(self, y, out=None):
        """Twofold ln(y0+y1) of a coupled twofold (tlogp, explog.py:239-242)."""
        return self._call("tlogp", y, out)

    def plog(self, y, out=None):
        """Pair ln(y0+y1) of a coupled twofold (plog, explog.py:251-258)."""
        return self._call("plog", y, out)

    def plog1p0(self, y, out=None):
        """Pair ln(1+y) of a plain y (plog1p0, explog.py:296-303)."""
        return self._call("plog1p0", y, out)

    def tlog1p0(self, y, out=None):
        """Twofold ln(1+y) of a plain y (tlog1p0, explog.py:305-308)."""
        return self._call("tlog1p0", y, out)

    def tlog1pp(self, y, out=None):
        """Twofold ln(1+y0+y1) of a coupled twofold (tlog1pp, explog.py:310-312)."""
        return self._call("tlog1pp", y, out)

    def plog1p(self, y, out=None):
        """Pair ln(1+y0+y1) of a coupled twofold (plog1p, explog.py:319-325)."""
        return self._call("plog1p", y, out)

    def function(self, name: str):
        if name not in FUNCTION_NAMES:
            raise ValueError(f"unknown function {name!r}")
        return getattr(self, name)

    # ---- dispatch
    def _call(self, fn: str, x, out=None):
        # one element on Python floats, the reference's own calling convention
        # (audit.py:343-349): straight to the small-call path
        tx = type(x)
        if tx is Twofold or tx is tuple:
            if (out is None and len(x) == 2 and type(x[0]) is float and type(x[1]) is float
                    and fn not in DOTTED_ARG):
                return self._scalar(fn, x[0], x[1])
        elif tx is float and out is None and fn in DOTTED_ARG:
            return self._scalar(fn, x, x)
        if fn in DOTTED_ARG:
            # plain argument: the kernel never reads x1, so alias it to x0
            if isinstance(x, Twofold) or isinstance(x, tuple):
                raise TypeError(f"{fn} takes a plain argument, not a twofold")
            x0 = x1 = x
        else:
            x0, x1 = x[0], x[1]
        if _is_torch(x0) or _is_torch(x1):
            if not (_is_torch(x0) and _is_torch(x1)):
                raise TypeError("both twofold parts must be torch tensors")
            if x0.is_cuda or x1.is_cuda:
                return self._device(fn, x0, x1, out)
            return self._host_torch(fn, x0, x1, out)
        if np.isscalar(x0) and np.isscalar(x1) or (isinstance(x0, (int, float)) and
                                                   isinstance(x1, (int, float))):
            return self._scalar(fn, x0, x1)
        a0 = np.asarray(x0)
        a1 = np.asarray(x1)
        if a0.shape != a1.shape:
            raise ValueError(f"twofold parts differ in shape: {a0.shape} vs {a1.shape}")
        z0, z1 = self._host_numpy(fn, a0.astype(self._np, copy=False),
                                  a1.astype(self._np, copy=False))
        return Twofold(z0, z1)

    def _scalar(self, fn, x0, x1):
        """One element, the reference's own calling convention (audit.py:343-349):
        straight through tf_eval_host's small-call path (operands in a mapped
        pinned buffer the tiny kernel reads over PCIe; one launch, then a spin on
        the completion flag the kernel stores after its results)."""
        L = _lib._lib or _lib.scalar_device()
        ct = self._ct
        z0, z1 = ct(), ct()
        # the device is the calling thread's current one (the library reads it
        # from the driver's current context, which torch.cuda.set_device sets);
        # stream NULL: the library's own non-blocking stream (host operands,
        # nothing on the device to order after).  No GPU: rc reports it.
        rc = L.tf_eval_host(_lib.FN_CODES[fn], self.width, byref(ct(x0)), byref(ct(x1)),
                            byref(z0), byref(z1), 1, 0, None, 0)
        if rc:
            _lib.scalar_device()          # raises "no CUDA device visible" first
            _lib.check(rc, f"tf_eval_host({fn}, width={self.width})")
        return Twofold(z0.value, z1.value)

    def _torch_dtype(self):
        import torch

        return torch.float64 if self.width == 64 else torch.float32

    def _launch(self, fn, x0, x1, z0, z1, n, stream_ptr, flags=0):
        L = _lib.ensure_device(x0.device.index if x0.device.index is not None else 0)
        rc = L.tf_eval(_lib.FN_CODES[fn], self.width, x0.data_ptr(), x1.data_ptr(),
                       z0.data_ptr(), z1.data_ptr(), n, stream_ptr, flags)
        _lib.check(rc, f"tf_eval({fn}, width={self.width})")

    def _device(self, fn, x0, x1, out=None, flags=0):
        import torch

        dt = self._torch_dtype()
        if x0.dtype != dt or x1.dtype != dt:
            raise TypeError(f"binary{self.width} twofolds need {dt} tensors, got "
                            f"{x0.dtype}/{x1.dtype}")
        if x0.shape != x1.shape:
            raise ValueError(f"twofold parts differ in shape: {tuple(x0.shape)} vs "
                             f"{tuple(x1.shape)}")
        if x0.device != x1.device:
            raise ValueError("twofold parts live on different devices")
        a0 = x0.contiguous()
        a1 = x1.contiguous()
        if out is None:
            z0 = torch.empty_like(a0)
            z1 = torch.empty_like(a1)
        else:
            z0, z1 = out
            if (z0.shape != a0.shape or z1.shape != a0.shape or z0.dtype != dt or
                    z1.dtype != dt or not z0.is_contiguous() or not z1.is_contiguous()):
                raise ValueError("out= tensors must be contiguous, same shape and dtype")
            if z0.device != a0.device or z1.device != a0.device:
                raise ValueError(f"out= tensors must live on the operands' device {a0.device}, "
                                 f"got {z0.device}/{z1.device}")
            # in place is supported element for element (z0 is x0 / z1 is x1: the
            # kernel's rare queue keeps the operands); any other overlap is not
            if _overlaps(z0, z1) or any(_overlaps(z, a) and not _same_span(z, a)
                                        for z in (z0, z1) for a in (a0, a1)):
                raise ValueError("out= tensors may alias the inputs only element for element")
        with torch.cuda.device(a0.device):
            stream = torch.cuda.current_stream(a0.device).cuda_stream
            self._launch(fn, a0, a1, z0, z1, a0.numel(), stream, flags)
        return Twofold(z0, z1)

    def _host_torch(self, fn, x0, x1, out=None):
        dt = self._torch_dtype()
        if x0.shape != x1.shape:
            raise ValueError(f"twofold parts differ in shape: {tuple(x0.shape)} vs "
                             f"{tuple(x1.shape)}")
        a0 = x0.to(dt).contiguous().reshape(-1)
        a1 = x1.to(dt).contiguous().reshape(-1)
        if out is not None:
            o0, o1 = out
            if (o0.shape != x0.shape or o1.shape != x0.shape or o0.dtype != dt or
                    o1.dtype != dt or o0.is_cuda or o1.is_cuda or not o0.is_contiguous()
                    or not o1.is_contiguous()):
                raise ValueError("out= host tensors must be contiguous CPU tensors of the "
                                 "input shape and lane dtype (pinned for full PCIe speed)")
            out = (o0.reshape(-1), o1.reshape(-1))
        z0, z1 = _pipeline(self, fn, a0, a1, out=out)
        return Twofold(z0.reshape(x0.shape), z1.reshape(x0.shape))

    def _host_numpy(self, fn, a0, a1):
        import torch

        t0 = torch.from_numpy(np.ascontiguousarray(a0).reshape(-1))
        t1 = torch.from_numpy(np.ascontiguousarray(a1).reshape(-1))
        z0, z1 = _pipeline(self, fn, t0, t1)
        return z0.numpy().reshape(a0.shape), z1.numpy().reshape(a0.shape)


def _pipeline(lib: ExpLog, fn: str, h0, h1, device=None, chunk: int = 0, out=None):
    """Evaluate host tensors through tf_eval_host (csrc/tf_host.cu): a three-stage
    chunk pipeline -- H2D, kernel and D2H on three streams over a ring of device
    buffers -- so both PCIe directions stay busy at once.  `out` may supply
    (pinned) host result tensors; otherwise pinned ones are allocated."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the twofold kernels need a B200 "
                           "(sm_100a); there is no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    n = h0.numel()
    dotted = fn in DOTTED_ARG
    if out is not None:
        z0, z1 = out
    else:
        z0 = torch.empty(n, dtype=h0.dtype, pin_memory=True)
        z1 = torch.empty(n, dtype=h0.dtype, pin_memory=True)
    if n == 0:
        return z0, z1
    if not h0.is_pinned():
        h0 = h0.pin_memory()
    if dotted:
        h1 = h0
    elif not h1.is_pinned():
        h1 = h1.pin_memory()
    L = _lib.ensure_device(dev.index)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = L.tf_eval_host(_lib.FN_CODES[fn], lib.width, h0.data_ptr(),
                            None if dotted else h1.data_ptr(), z0.data_ptr(), z1.data_ptr(),
                            n, chunk, stream, 0)
    _lib.check(rc, f"tf_eval_host({fn}, width={lib.width})")
    return z0, z1


@lru_cache(maxsize=None)
def _api_cached(width: int, backend: str) -> ExpLog:
    return ExpLog(width, backend)


def api(width: int, backend: str | None = None) -> ExpLog:
    """Cached function surface for (width, backend) (explog.py:338-344)."""
    if backend is None:
        backend = get_default_backend()
    elif backend not in ("fma", "dv"):
        raise ValueError(f"unknown backend {backend!r}")
    return _api_cached(width, backend)


def get_function(name: str, width: int, backend: str | None = None):
    """Resolve one of the twenty function names for a width (explog.py:347-349)."""
    return api(width, backend).function(name)

