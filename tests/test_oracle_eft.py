"""Pin the C restatement of the element-wise EFT / twofold arithmetic ops
(oracle/twofold_oracle.c tfo_eft) against outputs of the reference's own
eft.py / eft32.py (tests/golden/eft_golden.npz, made by
tests/golden/gen_eft_golden.py): bit for bit, both lanes, both residual
backends, thirteen ops; and the C-ABI argument checks of tf_eft (no GPU)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O
from oracle.compare import same_bits


@pytest.fixture(scope="module")
def eftg():
    return dict(np.load(os.path.join(GOLDEN, "eft_golden.npz")))


@pytest.mark.parametrize("backend", ("fma", "dv"))
@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("op", O.EFT_OPS)
def test_oracle_eft_matches_reference(op, width, backend, eftg):
    k = f"{op}_{width}_{backend}"
    z0, z1 = O.eft_arrays(op, width, eftg[k + "_a0"], eftg[k + "_a1"], eftg[k + "_b0"],
                          eftg[k + "_b1"], backend=backend)
    bad = ~(same_bits(z0, eftg[k + "_z0"]) & same_bits(z1, eftg[k + "_z1"]))
    assert not bad.any(), np.nonzero(bad)[0][:5]
    assert z0.size > 1000


def test_tf_eft_argument_errors():
    from paper_1502_05216_b200 import _lib

    L = _lib.load()
    assert L.tf_eft(0, 64, 0, None, None, None, None, None, None, 0, None) == 0
    assert L.tf_eft(13, 64, 0, 8, 8, 8, 8, 8, 8, 4, None) == _lib.TF_ERR_ARG
    assert b"op code" in L.tf_last_error()
    assert L.tf_eft(7, 64, 2, 8, 8, 8, 8, 8, 8, 4, None) == _lib.TF_ERR_ARG
    assert L.tf_eft(7, 16, 0, 8, 8, 8, 8, 8, 8, 4, None) == _lib.TF_ERR_ARG
    assert L.tf_eft(7, 64, 0, 8, 8, 8, None, 8, 8, 4, None) == _lib.TF_ERR_ARG   # t_add needs b1
    assert L.tf_eft(7, 64, 0, 8, 8, 8, 8, 8, 8, -1, None) == _lib.TF_ERR_ARG
    assert sorted(_lib.OP_CODES) == sorted(O.EFT_OPS)
    assert all(_lib.OP_CODES[n] == i for i, n in enumerate(O.EFT_OPS))
