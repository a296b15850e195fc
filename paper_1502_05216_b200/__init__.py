"""B200-native twofold exp/log: drop-in for the reference ``twofold`` package's
texp / texpm1 / tlog / tlog1p hot path (arXiv 1502.05216, E. Latkin).

    >>> import torch
    >>> from paper_1502_05216_b200 import api, Twofold
    >>> f64 = api(64)
    >>> x0 = torch.rand(1 << 20, dtype=torch.float64, device="cuda")
    >>> z = f64.texp(Twofold(x0, torch.zeros_like(x0)))   # z.value == exp(x0), CR

Re-exports follow the reference __init__.py:19-57.
"""

from .eft import SplitPair, Twofold, get_default_backend, set_default_backend
from .explog import (
    COUPLED_ARG,
    DOTTED_ARG,
    FAMILIES,
    FUNCTION_NAMES,
    TWOFOLD_ARG,
    ExpLog,
    api,
    family_of,
    get_function,
)

__version__ = "0.1.0"

# the kernels always use a hardware fused multiply-add for product residuals
HAVE_NATIVE_FMA = True


def assert_round_to_nearest() -> None:
    """Host-side rounding-mode probe (reference _fp.py:56-73); the kernels use
    explicit round-to-nearest intrinsics regardless of the host mode."""
    eps = 2.0 ** -53
    ok = (1.0 + eps == 1.0 and 1.0 + 3.0 * eps == 1.0 + 4.0 * eps
          and -1.0 - eps == -1.0 and -1.0 - 3.0 * eps == -1.0 - 4.0 * eps)
    if not ok:
        raise RuntimeError("floating-point rounding mode is not round-to-nearest-even; "
                           "refusing to run")


assert_round_to_nearest()

__all__ = [
    "Twofold", "SplitPair", "ExpLog", "api", "get_function", "family_of", "FAMILIES",
    "FUNCTION_NAMES", "DOTTED_ARG", "COUPLED_ARG", "TWOFOLD_ARG", "set_default_backend",
    "get_default_backend", "HAVE_NATIVE_FMA", "assert_round_to_nearest", "__version__",
]
