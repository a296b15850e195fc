"""GPU accuracy audit: the triple-double etalon
against mpmath, run_accuracy over all twenty functions at both widths against
the reference's own thresholds (audit.py:42-51), a negative control, the
binary32 library etalon, run_bench's checksum and run_demo."""

import math

import numpy as np
import pytest

from paper_1502_05216_b200 import FUNCTION_NAMES, audit

pytestmark = pytest.mark.gpu

FAMS = ("exp", "expm1", "log", "log1p")


def _etalon(fam, x0, x1, dev):
    import torch

    from paper_1502_05216_b200 import _lib

    L = _lib.ensure_device(dev.index)
    a0 = torch.from_numpy(np.ascontiguousarray(x0, np.float64)).to(dev)
    a1 = torch.from_numpy(np.ascontiguousarray(x1, np.float64)).to(dev)
    n = a0.numel()
    m = torch.empty(3 * n, dtype=torch.float64, device=dev)
    k = torch.empty(n, dtype=torch.int32, device=dev)
    _lib.check(L.tf_etalon(_lib.FAMILY_CODES[fam], a0.data_ptr(), a1.data_ptr(), n,
                           m.data_ptr(), k.data_ptr(), None), "tf_etalon")
    torch.cuda.synchronize()
    return m.cpu().numpy().reshape(3, n), k.cpu().numpy()


def _points(fam):
    """Audit-stream samples of both widths plus edges of every branch."""
    xs = []
    for w in (64, 32):
        name = {"exp": "texp", "expm1": "texpm1", "log": "tlog", "log1p": "tlog1p"}[fam]
        a0, a1 = audit.gen_sample_arrays(audit.SampleSpec(name, w, 600, 7))
        xs += list(zip(a0.astype(np.float64), a1.astype(np.float64)))
    edge = {"exp": [0.0, 1e-300, -1e-300, 0.34657, -0.34657, 0.5, 700.0, -740.0, 709.7, -708.4],
            "expm1": [1e-30, -1e-30, 0.339, 0.341, -0.339, -0.341, 0.7, -0.7, 30.0, -40.0],
            "log": [1.0, 1.0 + 2.0 ** -52, 1.0 - 2.0 ** -53, 0.70710678, 1.41421356, 2.0 ** -1000,
                    2.0 ** 1000, 3.0, 0.5, 1e-300],
            "log1p": [1e-30, -1e-30, 0.40999, 0.41001, -0.28999, -0.29001, -1.0 + 2.0 ** -52,
                      1e300, 5.0, -0.75]}[fam]
    xs += [(v, 0.0) for v in edge] + [(v, v * 2.0 ** -60) for v in edge]
    a = np.array(xs)
    return a[:, 0].copy(), a[:, 1].copy()


@pytest.mark.parametrize("fam", FAMS)
def test_etalon_against_mpmath(fam, cuda):
    import mpmath

    x0, x1 = _points(fam)
    m, k = _etalon(fam, x0, x1, cuda)
    f = {"exp": mpmath.exp, "expm1": mpmath.expm1, "log": mpmath.log, "log1p": mpmath.log1p}[fam]
    worst = 0.0
    with mpmath.workprec(260):
        for i in range(x0.size):
            ref = f(mpmath.mpf(float(x0[i])) + mpmath.mpf(float(x1[i])))
            got = (mpmath.mpf(float(m[0, i])) + mpmath.mpf(float(m[1, i])) +
                   mpmath.mpf(float(m[2, i]))) * mpmath.mpf(2) ** int(k[i])
            if ref == 0:
                assert got == 0, (x0[i], x1[i])
                continue
            rel = float(abs((got - ref) / ref))
            worst = max(worst, rel)
    print(fam, "worst etalon rel err 2^%.1f" % math.log2(worst + 1e-300))
    assert worst < 2.0 ** -135


@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("fn", FUNCTION_NAMES)
def test_audit_passes_reference_thresholds(fn, width, cuda):
    rep = audit.run_accuracy(audit.SampleSpec(fn, width, 50_000, 42))
    print(rep.summary_line())
    assert rep.passed, rep.summary_line()
    assert rep.subnormals_excluded < rep.samples // 2
    assert rep.l0_rel < 2.0 ** (-80 if width == 64 else -30)


def test_audit_negative_control(cuda):
    """A 2^-90 relative perturbation of the error part must fail the gate."""
    from paper_1502_05216_b200 import Twofold, api

    f = api(64).texp

    def bad(x):
        z = f(x)
        return Twofold(z.value, z.error + z.value * 2.0 ** -90)

    rep = audit.run_accuracy(audit.SampleSpec("texp", 64, 5_000, 3), fn_override=bad)
    assert not rep.passed and rep.l1_rel > 2.0 ** -92


@pytest.mark.parametrize("fn", ("texp", "texpm1", "tlog", "tlog1p"))
def test_lib_etalon_binary32(fn, cuda):
    rep = audit.run_accuracy(audit.SampleSpec(fn, 32, 20_000, 5), etalon="lib")
    assert rep.etalon == "lib"
    assert rep.l1_rel < 2.0 ** -40, rep.summary_line()


@pytest.mark.parametrize("width", (64, 32))
def test_bench_checksum(width, cuda):
    from paper_1502_05216_b200 import Twofold, api

    rep = audit.run_bench("tlog1p", width, 100_003)
    assert rep.iterations == 100_003 and rep.mops > 0 and rep.baseline_mops > 0
    spec = audit.SampleSpec("tlog1p", width, 1024, 0xB0B)
    x0, x1 = audit.gen_sample_arrays(spec)
    z = getattr(api(width), "tlog1p")(Twofold(x0, x1))
    bits = np.asarray(z.value, dtype=np.float64).view(np.uint64)
    counts = np.array([(100_003 - j + 1023) // 1024 for j in range(1024)])
    h = np.bitwise_xor.reduce(bits[counts % 2 == 1]) if (counts % 2).any() else np.uint64(0)
    assert rep.checksum == f"{int(h):016x}"


def test_demo(cuda):
    rep = audit.run_demo()
    assert rep.passed, rep.failures()
