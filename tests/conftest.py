import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
FNS = ("texp", "texpm1", "tlog", "tlog1p")
# the other sixteen names of FUNCTION_NAMES (reference explog.py:44-53)
SIBLINGS = ("pexp0", "texp0", "texpp", "pexp", "pexpm10", "texpm10", "texpm1p", "pexpm1",
            "plog0", "tlog0", "tlogp", "plog", "plog1p0", "tlog1p0", "tlog1pp", "plog1p")
ALL_FNS = FNS + SIBLINGS


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(fn, width):
        key = (fn, width)
        if key not in cache:
            cache[key] = dict(np.load(os.path.join(GOLDEN, f"golden_{fn}_f{width}.npz")))
        return cache[key]

    return load


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1502_05216_b200 import _lib

    _lib.ensure_device(torch.cuda.current_device())
    return torch.device("cuda", torch.cuda.current_device())
