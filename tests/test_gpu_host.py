"""Host-buffer entry point (tf_eval_host, csrc/tf_host.cu): the reference's own
calling convention -- api(width) methods on host arrays (explog.py:333-349) --
through the three-stream chunk pipeline.  Every result must be bit-identical
to the device-pointer path on the same inputs, for any chunk size (ring
wrap-around, ragged last chunk), pinned or pageable memory, numpy or torch
host arrays, and dotted functions with x1 = NULL."""

import numpy as np
import pytest

from conftest import ALL_FNS, FNS

pytestmark = pytest.mark.gpu


def _inputs(fn, width, n, seed=7):
    rng = np.random.default_rng(seed)
    dt = np.float64 if width == 64 else np.float32
    if fn.startswith(("texp", "pexp")):
        x0 = rng.uniform(-30.0, 30.0, n)
    else:
        x0 = np.exp(rng.uniform(-20.0, 20.0, n)) - (0.5 if "1p" in fn else 0.0)
    x0 = x0.astype(dt)
    x1 = (x0.astype(np.float64) * rng.uniform(-1, 1, n) * 2.0 ** (-53 if width == 64 else -24))
    return x0, x1.astype(dt)


def _device_ref(fn, width, x0, x1):
    import torch

    from paper_1502_05216_b200 import api

    t0, t1 = torch.from_numpy(x0).cuda(), torch.from_numpy(x1).cuda()
    f = getattr(api(width), fn)
    z = f(t0) if fn.endswith("0") else f((t0, t1))
    torch.cuda.synchronize()
    return z.value.cpu().numpy(), z.error.cpu().numpy()


def _host(fn, width, x0, x1, chunk, pinned=True):
    import torch

    from paper_1502_05216_b200 import _lib

    L = _lib.ensure_device(0)
    h0, h1 = torch.from_numpy(x0.copy()), torch.from_numpy(x1.copy())
    z0, z1 = torch.empty_like(h0), torch.empty_like(h0)
    if pinned:
        h0, h1, z0, z1 = (t.pin_memory() for t in (h0, h1, z0, z1))
    dotted = fn.endswith("0")
    rc = L.tf_eval_host(_lib.FN_CODES[fn], width, h0.data_ptr(), None if dotted else h1.data_ptr(),
                        z0.data_ptr(), z1.data_ptr(), x0.size, chunk, None, 0)
    _lib.check(rc, "tf_eval_host")
    return z0.numpy(), z1.numpy()


@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("fn", FNS)
@pytest.mark.parametrize("chunk", (0, 1, 1000, 4099, 1 << 20))
def test_host_pipeline_equals_device_path(fn, width, chunk, cuda):
    n = 3 if chunk == 1 else 10007          # chunk 1 wraps the 4-slot ring
    x0, x1 = _inputs(fn, width, n)
    r0, r1 = _device_ref(fn, width, x0, x1)
    z0, z1 = _host(fn, width, x0, x1, chunk)
    np.testing.assert_array_equal(z0.view(np.uint8), r0.view(np.uint8))
    np.testing.assert_array_equal(z1.view(np.uint8), r1.view(np.uint8))


@pytest.mark.parametrize("fn", [f for f in ALL_FNS if f not in FNS])
def test_host_pipeline_siblings(fn, cuda):
    x0, x1 = _inputs(fn, 64, 5000, seed=11)
    if fn.endswith("0"):
        x1 = np.zeros_like(x1)
    r0, r1 = _device_ref(fn, 64, x0, x1)
    z0, z1 = _host(fn, 64, x0, x1, 777)
    np.testing.assert_array_equal(z0.view(np.uint8), r0.view(np.uint8))
    np.testing.assert_array_equal(z1.view(np.uint8), r1.view(np.uint8))


def test_host_pipeline_pageable_memory(cuda):
    x0, x1 = _inputs("tlog1p", 64, 300001)
    r0, r1 = _device_ref("tlog1p", 64, x0, x1)
    z0, z1 = _host("tlog1p", 64, x0, x1, 65536, pinned=False)
    np.testing.assert_array_equal(z0.view(np.uint8), r0.view(np.uint8))
    np.testing.assert_array_equal(z1.view(np.uint8), r1.view(np.uint8))


@pytest.mark.parametrize("width", (64, 32))
def test_public_api_on_host_arrays(width, cuda):
    """numpy in / numpy out and torch CPU in / CPU out (with out=) both run
    through tf_eval_host and agree with the device path."""
    import torch

    from paper_1502_05216_b200 import Twofold, api

    x0, x1 = _inputs("texpm1", width, (1 << 20) + 3)
    r0, r1 = _device_ref("texpm1", width, x0, x1)
    z = api(width).texpm1((x0, x1))
    assert isinstance(z.value, np.ndarray)
    np.testing.assert_array_equal(z.value.view(np.uint8), r0.view(np.uint8))
    np.testing.assert_array_equal(z.error.view(np.uint8), r1.view(np.uint8))
    h0, h1 = torch.from_numpy(x0).pin_memory(), torch.from_numpy(x1).pin_memory()
    o0, o1 = torch.empty_like(h0).pin_memory(), torch.empty_like(h0).pin_memory()
    z = api(width).texpm1(Twofold(h0, h1), out=(o0, o1))
    assert z.value.data_ptr() == o0.data_ptr() and not z.value.is_cuda
    np.testing.assert_array_equal(o0.numpy().view(np.uint8), r0.view(np.uint8))
    np.testing.assert_array_equal(o1.numpy().view(np.uint8), r1.view(np.uint8))


def test_host_pipeline_orders_after_caller_stream(cuda):
    """Pinned input written by a device->host copy still queued on the caller's
    stream: tf_eval_host must read it only after that copy lands."""
    import torch

    from paper_1502_05216_b200 import _lib

    n = 1 << 22
    x0, x1 = _inputs("tlog", 64, n)
    r0, r1 = _device_ref("tlog", 64, x0, x1)
    s = torch.cuda.Stream()
    d0 = torch.from_numpy(x0).cuda()
    h0 = torch.zeros(n, dtype=torch.float64).pin_memory()
    h1 = torch.from_numpy(x1).pin_memory()
    z0, z1 = torch.empty_like(h0).pin_memory(), torch.empty_like(h0).pin_memory()
    L = _lib.ensure_device(0)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(20_000_000)        # keep the caller's stream busy
        h0.copy_(d0, non_blocking=True)
        rc = L.tf_eval_host(_lib.FN_CODES["tlog"], 64, h0.data_ptr(), h1.data_ptr(),
                            z0.data_ptr(), z1.data_ptr(), n, 0, s.cuda_stream, 0)
    _lib.check(rc, "tf_eval_host")
    np.testing.assert_array_equal(z0.numpy().view(np.uint8), r0.view(np.uint8))
    np.testing.assert_array_equal(z1.numpy().view(np.uint8), r1.view(np.uint8))


def test_host_pipeline_concurrent_callers(cuda):
    """Calls from several host threads at once take different pipelines of the
    per-device pool (or queue on a busy one): every result equals the
    device-pointer path bit for bit."""
    from concurrent.futures import ThreadPoolExecutor

    import torch

    jobs = [(fn, 64 if k % 2 == 0 else 32, k) for k, fn in enumerate(FNS * 2)]
    data = {j: _inputs(j[0], j[1], 300_001 + 17 * j[2], seed=j[2]) for j in jobs}

    def run(j):
        torch.cuda.set_device(cuda)
        return _host(j[0], j[1], *data[j], chunk=1 << 16)

    with ThreadPoolExecutor(4) as pool:
        got = list(pool.map(run, jobs))
    for j, (z0, z1) in zip(jobs, got):
        r0, r1 = _device_ref(j[0], j[1], *data[j])
        assert np.array_equal(z0.view(np.uint8), r0.view(np.uint8)), j
        assert np.array_equal(z1.view(np.uint8), r1.view(np.uint8)), j


@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("fn", FNS)
def test_scalar_calls_equal_array_calls(fn, width, cuda):
    """Python-float calls (the reference's convention) take tf_eval_host's
    small-call path (mapped pinned buffer); results equal the device path."""
    import numpy as np

    from paper_1502_05216_b200 import api

    x0, x1 = _inputs(fn, width, 64)
    z0, z1 = _device_ref(fn, width, x0, x1)
    f = getattr(api(width), fn)
    for i in range(64):
        r = f((float(x0[i]), float(x1[i])))
        assert np.array([r.value], dtype=x0.dtype).view(np.uint8).tobytes() == \
            z0[i:i + 1].view(np.uint8).tobytes()
        same1 = np.array([r.error], dtype=x0.dtype).view(np.uint8).tobytes() == \
            z1[i:i + 1].view(np.uint8).tobytes()
        assert same1 or (np.isnan(r.error) and np.isnan(z1[i]))


@pytest.mark.parametrize("width", (64, 32))
def test_scalar_twofold_dotted_and_thread_calls(width, cuda):
    """The reference's own scalar forms -- a Twofold of Python floats, a plain
    float for the dotted functions (audit.py:334-349) -- and calls from a
    second host thread all equal the device path bit for bit."""
    import threading

    import numpy as np

    from paper_1502_05216_b200 import Twofold, api

    lib = api(width)
    x0, x1 = _inputs("texp", width, 16)
    z0, z1 = _device_ref("texp", width, x0, x1)
    d0, d1 = _device_ref("texp0", width, x0, np.zeros_like(x0))
    got = {}

    def run(key):
        got[key] = [(lib.texp(Twofold(float(x0[i]), float(x1[i]))), lib.texp0(float(x0[i])))
                    for i in range(16)]

    run("main")
    t = threading.Thread(target=run, args=("thread",))
    t.start()
    t.join()
    for key, res in got.items():
        for i, (r, r0) in enumerate(res):
            assert np.array([r.value, r.error], dtype=x0.dtype).tobytes() == \
                np.array([z0[i], z1[i]], dtype=x0.dtype).tobytes(), (key, i)
            assert np.array([r0.value, r0.error], dtype=x0.dtype).tobytes() == \
                np.array([d0[i], d1[i]], dtype=x0.dtype).tobytes(), (key, i)


def test_small_host_arrays_use_mapped_path(cuda):
    """n <= 1024 host arrays go through the small-call path; results equal the
    chunked pipeline's bit for bit."""
    import numpy as np

    for n in (1, 7, 1024):
        x0, x1 = _inputs("tlog", 64, n)
        a = _host("tlog", 64, x0, x1, chunk=0)
        b = _host("tlog", 64, x0, x1, chunk=3)
        assert np.array_equal(a[0].view(np.int64), b[0].view(np.int64))
        assert np.array_equal(a[1].view(np.int64), b[1].view(np.int64))
