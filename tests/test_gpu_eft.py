"""GPU element-wise EFTs / twofold arithmetic (csrc/tf_eft.cu) against outputs
of the reference's eft.py / eft32.py (golden vectors), through the public
Python surface (eft / eft32 free functions and arith bundles), and against the
C oracle at 2^20 random elements per op."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O
from oracle.compare import same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eftg():
    return dict(np.load(os.path.join(GOLDEN, "eft_golden.npz")))


def _call(op, width, backend, a0, a1, b0, b1):
    from paper_1502_05216_b200 import Twofold, eft, eft32

    mod = eft if width == 64 else eft32
    ar = mod.arith(backend)
    x, y = Twofold(a0, a1), Twofold(b0, b1)
    f = {
        "fast_two_sum": lambda: mod.fast_two_sum(a0, b0),
        "two_sum": lambda: mod.two_sum(a0, b0),
        "two_diff": lambda: mod.two_diff(a0, b0),
        "two_prod": lambda: (mod.two_prod_fma if backend == "fma" else mod.two_prod_dv)(a0, b0),
        "split": lambda: mod.split(a0),
        "renorm_fast": lambda: mod.renorm_fast(x),
        "renorm": lambda: mod.renorm(x),
        "t_add": lambda: ar.t_add(x, y),
        "t_add_d": lambda: ar.t_add_d(x, b0),
        "t_mul": lambda: ar.t_mul(x, y),
        "t_mul_d": lambda: ar.t_mul_d(x, b0),
        "t_div": lambda: ar.t_div(x, y),
        "t_sqrt": lambda: ar.t_sqrt(x),
    }[op]
    return f()


@pytest.mark.parametrize("backend", ("fma", "dv"))
@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("op", O.EFT_OPS)
def test_eft_ops_match_reference(op, width, backend, eftg, cuda):
    import torch

    k = f"{op}_{width}_{backend}"
    args = [torch.from_numpy(eftg[k + s]).to(cuda) for s in ("_a0", "_a1", "_b0", "_b1")]
    r = _call(op, width, backend, *args)
    z0, z1 = r[0].cpu().numpy(), r[1].cpu().numpy()
    bad = ~(same_bits(z0, eftg[k + "_z0"]) & same_bits(z1, eftg[k + "_z1"]))
    assert not bad.any(), [(eftg[k + "_a0"][i], eftg[k + "_b0"][i]) for i in np.nonzero(bad)[0][:3]]


@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("op", O.EFT_OPS)
def test_eft_ops_large_vs_oracle(op, width, cuda):
    import torch

    from paper_1502_05216_b200 import _lib

    rng = np.random.default_rng(11 + width)
    n = (1 << 20) + 5
    dt = np.float64 if width == 64 else np.float32
    e = rng.integers(-60, 60, (4, n))
    v = (rng.uniform(1, 2, (4, n)) * rng.choice([-1, 1], (4, n)) * np.exp2(e)).astype(dt)
    v[1] = (v[0].astype(np.float64) * rng.uniform(-1, 1, n) * 2.0 ** -(53 if width == 64 else 24)).astype(dt)
    v[3] = (v[2].astype(np.float64) * rng.uniform(-1, 1, n) * 2.0 ** -(53 if width == 64 else 24)).astype(dt)
    if op == "t_sqrt":
        v[0] = np.abs(v[0])
    L = _lib.ensure_device(cuda.index)
    for backend in ("fma", "dv"):
        t = [torch.from_numpy(a).to(cuda) for a in v]
        z0, z1 = torch.empty_like(t[0]), torch.empty_like(t[0])
        _lib.check(L.tf_eft(_lib.OP_CODES[op], width, 1 if backend == "dv" else 0,
                            *[a.data_ptr() for a in t], z0.data_ptr(), z1.data_ptr(), n, None),
                   "tf_eft")
        torch.cuda.synchronize()
        r0, r1 = O.eft_arrays(op, width, *v, backend=backend)
        bad = ~(same_bits(z0.cpu().numpy(), r0) & same_bits(z1.cpu().numpy(), r1))
        assert not bad.any(), (backend, np.nonzero(bad)[0][:3])


def test_eft_scalar_and_host_inputs(cuda):
    from paper_1502_05216_b200 import Twofold, eft, eft32

    r = eft.two_sum(1.0, 2.0 ** -60)
    assert r == (1.0, 2.0 ** -60) and isinstance(r.value, float)
    h = eft.split(np.array([3.0, 134217729.0 * 3]))
    assert isinstance(h.hi, np.ndarray) and np.all(h.hi + h.lo == [3.0, 134217729.0 * 3])
    q = eft32.t_add(Twofold(1.0, 0.0), Twofold(2.0 ** -30, 0.0))
    assert q.value == 1.0 and q.error == 2.0 ** -30
    assert eft.arith("dv").backend == "dv"
    with pytest.raises(ValueError):
        eft.arith("x87")
    d = eft.t_div(Twofold(1.0, 0.0), Twofold(3.0, 0.0))
    assert d.value == 1.0 / 3.0 and abs(d.error) < 2.0 ** -54
    ar = eft.arith("fma")
    assert ar.prod_err(3.0, 1.0 / 3.0, 3.0 * (1.0 / 3.0)) == eft.two_prod_fma(3.0, 1.0 / 3.0).error
    from fractions import Fraction

    exact = Fraction(1) - 3 * Fraction(d.value)                # representable here
    assert ar.rem(d.value, 3.0, 1.0) == float(exact)
    assert eft.arith("dv").rem(d.value, 3.0, 1.0) == float(exact)
