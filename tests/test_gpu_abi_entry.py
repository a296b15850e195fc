"""GPU tests of the C-ABI surface itself (include/twofold_b200.h):

* the eight named batch entry points tf_{texp,texpm1,tlog,tlog1p}_f{64,32}
  (SURVEY.md 8(b)), called directly through ctypes on config samples, must
  equal tf_eval bit for bit and pass the oracle gate;
* in-place evaluation (z aliasing x element for element, the header's
  promise) must equal the out-of-place result bit for bit, including the
  rare elements the exact path re-evaluates (specials, FORCE_EXACT);
* one process may evaluate on several devices (the dynamic shared-memory
  attribute is per device): skipped with fewer than two GPUs.
"""

import ctypes

import numpy as np
import pytest

from conftest import ALL_FNS, FNS
from oracle import oracle as O
from oracle.compare import compare

pytestmark = pytest.mark.gpu

CFG_DIST = {("texp", 64): "exp64s", ("texpm1", 64): "pow10_64", ("tlog", 64): "logu64s",
            ("tlog1p", 64): "pow10c_64", ("texp", 32): "exp32", ("texpm1", 32): "exp32",
            ("tlog", 32): "log32", ("tlog1p", 32): "log32"}


def _dev_arrays(x0, x1, dev):
    import torch

    return (torch.from_numpy(np.ascontiguousarray(x0)).to(dev),
            torch.from_numpy(np.ascontiguousarray(x1)).to(dev))


@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("fn", FNS)
def test_named_entry_points(fn, width, cuda):
    import torch

    from paper_1502_05216_b200 import _lib, workloads

    L = _lib.load()
    x0, x1 = workloads.generate(CFG_DIST[(fn, width)], 123, 1 << 16, seed=5)
    a0, a1 = _dev_arrays(x0, x1, cuda)
    z0, z1 = torch.empty_like(a0), torch.empty_like(a0)
    e0, e1 = torch.empty_like(a0), torch.empty_like(a0)
    s = torch.cuda.current_stream(cuda).cuda_stream
    entry = getattr(L, f"tf_{fn}_f{width}")
    _lib.check(entry(a0.data_ptr(), a1.data_ptr(), z0.data_ptr(), z1.data_ptr(), a0.numel(), s),
               f"tf_{fn}_f{width}")
    _lib.check(L.tf_eval(_lib.FN_CODES[fn], width, a0.data_ptr(), a1.data_ptr(), e0.data_ptr(),
                         e1.data_ptr(), a0.numel(), s, 0), "tf_eval")
    torch.cuda.synchronize()
    assert torch.equal(z0.view(torch.int64 if width == 64 else torch.int32),
                       e0.view(torch.int64 if width == 64 else torch.int32))
    assert torch.equal(z1.view(torch.int64 if width == 64 else torch.int32),
                       e1.view(torch.int64 if width == 64 else torch.int32))
    r = O.evaluate(fn, width, x0, x1, backend="fma",
                   **({"libm64": "cr"} if width == 64 else {"libm32": "cr"}))
    c = compare(z0.cpu().numpy(), z1.cpu().numpy(), *r, width)
    assert c["class_mismatch"] == 0 and c["tol_violations"] == 0, c
    if width == 64:
        assert c["z0_gt1ulp"] == 0, c
    # argument errors come back as TF_ERR_ARG with a message, never an exception
    assert entry(a0.data_ptr(), a1.data_ptr(), z0.data_ptr(), z1.data_ptr(), -1, s) == _lib.TF_ERR_ARG
    assert entry(None, a1.data_ptr(), z0.data_ptr(), z1.data_ptr(), 4, s) == _lib.TF_ERR_ARG
    assert b"null" in L.tf_last_error()


@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("fn", ALL_FNS)
@pytest.mark.parametrize("force", (False, True))
def test_in_place_equals_out_of_place(fn, width, force, golden, cuda):
    """out=(x0, x1): the fast path overwrites elements that the rare queue
    re-evaluates later; the queue must carry the original operands."""
    from paper_1502_05216_b200 import _lib, api

    g = golden(fn, width)
    x0, x1 = g["x0"], g["x1"]
    dotted = fn.endswith("0")
    if dotted:
        x1 = np.zeros_like(x0)
    lib = api(width)
    flags = _lib.FLAG_FORCE_EXACT if force else 0
    a0, a1 = _dev_arrays(x0, x1, cuda)
    ref = lib._device(fn, a0, a1, flags=flags)
    b0, b1 = _dev_arrays(x0, x1, cuda)
    got = lib._device(fn, b0, b1, out=(b0, b1), flags=flags)
    assert got.value.data_ptr() == b0.data_ptr()
    r = compare(b0.cpu().numpy(), b1.cpu().numpy(), ref.value.cpu().numpy(),
                ref.error.cpu().numpy(), width)
    assert r["z0_mismatch"] == 0 and r["z1_bit_mismatch"] == 0, r


@pytest.mark.parametrize("fn", ("texp", "tlog"))
def test_in_place_config5_with_specials(fn, cuda):
    """BASELINE configs[4] inputs (1% specials) evaluated in place."""
    import torch

    from paper_1502_05216_b200 import api, workloads

    dist = "exp64s" if fn == "texp" else "logu64s"
    x0, x1 = workloads.generate(dist, 0, (1 << 20) + 7, seed=2024)
    a0, a1 = _dev_arrays(x0, x1, cuda)
    ref = getattr(api(64), fn)((a0, a1))
    b0, b1 = _dev_arrays(x0, x1, cuda)
    getattr(api(64), fn)((b0, b1), out=(b0, b1))
    torch.cuda.synchronize()
    assert torch.equal(b0.view(torch.int64), ref.value.view(torch.int64))
    assert torch.equal(b1.view(torch.int64), ref.error.view(torch.int64))


def test_out_tensors_on_wrong_device_rejected(cuda):
    import torch

    from paper_1502_05216_b200 import api

    a0 = torch.ones(8, dtype=torch.float64, device=cuda)
    a1 = torch.zeros(8, dtype=torch.float64, device=cuda)
    with pytest.raises(ValueError):
        api(64).texp((a0, a1), out=(torch.empty(8, dtype=torch.float64), torch.empty_like(a0)))
    buf = torch.ones(16, dtype=torch.float64, device=cuda)
    with pytest.raises(ValueError):          # partial overlap with the input
        api(64).texp((buf[:8], a1), out=(buf[4:12], torch.empty_like(a0)))
    with pytest.raises(ValueError):          # the two outputs overlap
        api(64).texp((a0, a1), out=(buf[:8], buf[2:10]))


def test_two_devices_one_process():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    from paper_1502_05216_b200 import api, workloads

    x0, x1 = workloads.generate("logu64s", 0, 1 << 18, seed=3)
    outs = []
    for d in (0, 1, 0):
        dev = torch.device("cuda", d)
        a0, a1 = _dev_arrays(x0, x1, dev)
        z = api(64).tlog((a0, a1))
        torch.cuda.synchronize(dev)
        outs.append((z.value.cpu(), z.error.cpu()))
    for v, e in outs[1:]:
        assert torch.equal(v.view(torch.int64), outs[0][0].view(torch.int64))
        assert torch.equal(e.view(torch.int64), outs[0][1].view(torch.int64))


def test_named_entry_point_scalar_c_form(cuda):
    """The paper's scalar C form z0 = texp(x0, x1, &z1) is the
    n == 1 case of tf_texp_f64."""
    import torch

    from paper_1502_05216_b200 import _lib

    L = _lib.load()
    a = torch.tensor([1.0], dtype=torch.float64, device=cuda)
    b = torch.tensor([2.0 ** -60], dtype=torch.float64, device=cuda)
    z0, z1 = torch.empty_like(a), torch.empty_like(a)
    _lib.check(L.tf_texp_f64(a.data_ptr(), b.data_ptr(), z0.data_ptr(), z1.data_ptr(), 1,
                             ctypes.c_void_p(0)), "tf_texp_f64")
    torch.cuda.synchronize()
    r0, r1 = O.evaluate("texp", 64, np.array([1.0]), np.array([2.0 ** -60]), backend="fma",
                        libm64="cr")
    assert z0.item() == r0[0] and z1.item() == r1[0]


@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("fn", ALL_FNS)
def test_tiny_launch_equals_full_kernel(fn, width, golden, cuda):
    """n <= 32 runs the one-warp k_tiny (the same fast path and rare-element
    sequence at one lane per thread, tables in global memory); every 32-element
    window of the golden vectors must equal the admission-band
    kernel's result on the whole array bit for bit."""
    from paper_1502_05216_b200 import api

    g = golden(fn, width)
    x0, x1 = g["x0"], g["x1"]
    if fn.endswith("0"):
        x1 = np.zeros_like(x0)
    lib = api(width)
    a0, a1 = _dev_arrays(x0, x1, cuda)
    full = lib._device(fn, a0, a1)
    f0, f1 = full.value.cpu().numpy(), full.error.cpu().numpy()
    for lo_ in range(0, min(x0.size, 32 * 24), 32):
        t0, t1 = _dev_arrays(x0[lo_:lo_ + 32], x1[lo_:lo_ + 32], cuda)
        z = lib._device(fn, t0, t1)
        r = compare(z.value.cpu().numpy(), z.error.cpu().numpy(), f0[lo_:lo_ + 32],
                    f1[lo_:lo_ + 32], width)
        assert r["z0_mismatch"] == 0 and r["z1_bit_mismatch"] == 0, (lo_, r)
