"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/twofold_b200.h declares, argument errors come back as
status codes without touching a GPU, and the Python surface mirrors the
reference package (pkg/src/twofold/explog.py:44-62, 333-349; __init__.py)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "twofold_b200.h")


def test_library_exports_header_symbols():
    from paper_1502_05216_b200 import _lib

    L = _lib.load()
    declared = re.findall(r"TF_API\s+[\w\s\*]+?\b(tf_\w+)\s*\(", open(HEADER).read())
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.tf_version() == 1


def test_library_is_sm100a():
    import subprocess

    from paper_1502_05216_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_argument_errors_without_gpu():
    from paper_1502_05216_b200 import _lib

    L = _lib.load()
    assert L.tf_eval(0, 64, None, None, None, None, 0, None, 0) == 0       # n == 0: no-op
    assert L.tf_eval(0, 64, None, None, None, None, -1, None, 0) == _lib.TF_ERR_ARG
    assert b"negative" in L.tf_last_error()
    assert L.tf_eval(0, 64, None, None, None, None, 5, None, 0) == _lib.TF_ERR_ARG
    assert b"null" in L.tf_last_error()
    assert L.tf_eval(0, 16, 8, 8, 8, 8, 5, None, 0) == _lib.TF_ERR_ARG
    assert L.tf_eval(20, 64, 8, 8, 8, 8, 5, None, 0) == _lib.TF_ERR_ARG     # TF_FN_COUNT
    assert L.tf_eval(-1, 32, 8, 8, 8, 8, 5, None, 0) == _lib.TF_ERR_ARG
    assert b"unknown function" in L.tf_last_error()
    # a plain-argument (dotted) function accepts x1 == NULL, the others do not
    assert L.tf_eval(_lib.FN_CODES["tlog"], 64, 8, None, 8, 8, 5, None, 0) == _lib.TF_ERR_ARG
    assert L.tf_texp_f64(None, None, None, None, 0, None) == 0
    assert L.tf_generate(99, 0, 0, 10, 8, 8, None) == _lib.TF_ERR_ARG
    assert L.tf_exact_count(None, 0) == _lib.TF_ERR_ARG
    # host-buffer entry point: argument checks precede any CUDA call
    assert L.tf_eval_host(0, 64, None, None, None, None, 0, 0, None, 0) == 0   # n == 0: no-op
    assert L.tf_eval_host(0, 64, 8, 8, 8, 8, -1, 0, None, 0) == _lib.TF_ERR_ARG
    assert L.tf_eval_host(0, 16, 8, 8, 8, 8, 5, 0, None, 0) == _lib.TF_ERR_ARG
    assert L.tf_eval_host(20, 64, 8, 8, 8, 8, 5, 0, None, 0) == _lib.TF_ERR_ARG
    assert L.tf_eval_host(0, 64, 8, 8, 8, 8, 5, -4, None, 0) == _lib.TF_ERR_ARG
    assert b"chunk" in L.tf_last_error()
    assert L.tf_eval_host(_lib.FN_CODES["tlog"], 64, 8, None, 8, 8, 5, 0, None, 0) == _lib.TF_ERR_ARG
    assert b"null" in L.tf_last_error()
    with pytest.raises(ValueError):
        _lib.check(-1, "x")


def test_api_surface_matches_reference():
    import paper_1502_05216_b200 as P

    assert P.FAMILIES == {
        "exp": ("pexp0", "texp0", "texp", "texpp", "pexp"),
        "expm1": ("pexpm10", "texpm10", "texpm1", "texpm1p", "pexpm1"),
        "log": ("plog0", "tlog0", "tlogp", "tlog", "plog"),
        "log1p": ("plog1p0", "tlog1p0", "tlog1pp", "tlog1p", "plog1p"),
    }
    assert len(P.FUNCTION_NAMES) == 20
    assert P.TWOFOLD_ARG == frozenset(("texp", "texpm1", "tlog", "tlog1p"))
    assert P.family_of("tlog1p") == "log1p"
    with pytest.raises(ValueError):
        P.family_of("sin")
    f = P.api(64)
    assert f is P.api(64) and f.width == 64 and f.backend in ("fma", "dv")
    assert f.params.N_exp == 12 and P.api(32).params.N_exp == 6
    assert P.api(64, "dv").backend == "dv"
    with pytest.raises(ValueError):
        P.api(16)
    with pytest.raises(ValueError):
        P.api(64, "avx")
    with pytest.raises(ValueError):
        P.get_function("nope", 64)
    assert P.get_function("texp", 64) == f.texp
    for name in P.FUNCTION_NAMES:                  # all twenty are served
        assert P.get_function(name, 32) == getattr(P.api(32), name)
    assert sorted(_codes()) == sorted(P.FUNCTION_NAMES)
    t = P.Twofold(1.0, 2.0)
    assert t.value == 1.0 and t.error == 2.0
    P.assert_round_to_nearest()


def _codes():
    from paper_1502_05216_b200 import _lib

    assert sorted(_lib.FN_CODES.values()) == list(range(20))
    return _lib.FN_CODES


def test_function_codes_match_header():
    """_lib.FN_CODES mirrors the TF_FN_* macros of include/twofold_b200.h."""
    import os
    import re

    from paper_1502_05216_b200 import _lib

    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "twofold_b200.h")).read()
    macros = {m.group(1).lower(): int(m.group(2))
              for m in re.finditer(r"#define TF_FN_([A-Z0-9]+) (\d+)", hdr)}
    assert macros.pop("count") == 20
    assert macros == _lib.FN_CODES


def test_backend_default_roundtrip():
    import paper_1502_05216_b200 as P

    old = P.get_default_backend()
    try:
        P.set_default_backend("dv")
        assert P.get_default_backend() == "dv"
    finally:
        P.set_default_backend(old)
    with pytest.raises(ValueError):
        P.set_default_backend("x")


def test_no_cpu_fallback():
    """The product path fails loudly without a GPU (no silent oracle use)."""
    import torch

    import paper_1502_05216_b200 as P

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        P.api(64).texp((1.0, 0.0))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        P.api(32).tlog((np.ones(4, np.float32), np.zeros(4, np.float32)))


def test_shape_and_type_errors():
    import torch

    import paper_1502_05216_b200 as P

    with pytest.raises(ValueError):
        P.api(64).texp((np.ones(3), np.ones(4)))
    with pytest.raises(TypeError):
        P.api(64).texp((torch.ones(3), np.ones(3)))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1502_05216_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "tforacle" not in text, f


def test_workloads_shard_invariant():
    from paper_1502_05216_b200 import workloads

    for dist in workloads.DISTS:
        a0, a1 = workloads.generate(dist, 0, 1000, seed=5)
        b0, b1 = workloads.generate(dist, 400, 600, seed=5)
        u = np.uint32 if a0.dtype == np.float32 else np.uint64
        assert np.array_equal(a0[400:].view(u), b0.view(u))
        assert np.array_equal(a1[400:].view(u), b1.view(u))


def test_workload_distributions():
    from paper_1502_05216_b200 import workloads

    x0, x1 = workloads.generate("exp64", 0, 100000, seed=1)
    assert -700 <= x0.min() and x0.max() <= 700
    assert np.all(np.abs(x1) <= np.abs(x0) * 2.0 ** -53)
    x0, _ = workloads.generate("pow10c_64", 0, 200000, seed=1)
    assert x0.min() >= -1.0 + 2.0 ** -52
    frac = np.mean(x0 == -1.0 + 2.0 ** -52)
    assert 0.0005 < frac < 0.004            # ~0.17% sit at the clamp
    x0, _ = workloads.generate("log64", 0, 200000, seed=1)
    assert 0.04 < np.mean(np.abs(x0 - 1.0) <= 2.0 ** -40) < 0.06
    x0, x1 = workloads.generate("exp64s", 0, 200000, seed=1)
    sp = np.isin(x0, workloads.SPECIALS_EXP64) | np.isnan(x0)
    assert 0.007 < np.mean(sp) < 0.013
    x0, _ = workloads.generate("log32", 0, 1000, seed=1)
    assert x0.dtype == np.float32 and x0.min() > 0


def test_compare_rules():
    from oracle.compare import compare

    one = np.array([1.0, np.inf, np.nan])
    r = compare(one, np.array([1e-17, np.inf, np.nan]), one, np.array([1e-17, np.inf, np.nan]), 64)
    assert r["z0_mismatch"] == 0 and r["tol_violations"] == 0 and r["class_mismatch"] == 0
    z0 = np.array([1.0])
    r = compare(np.nextafter(z0, 2), np.array([-2.0 ** -52]), z0, np.array([0.0]), 64)
    assert r["z0_mismatch"] == 1 and r["z0_gt1ulp"] == 0 and r["tol_violations"] == 0
    r = compare(z0, np.array([2.0 ** -80]), z0, np.array([0.0]), 64)
    assert r["tol_violations"] == 1
    r = compare(z0, np.array([np.inf]), z0, np.array([1e-17]), 64)
    assert r["class_mismatch"] == 1


def test_ctypes_pointer_argtypes():
    from paper_1502_05216_b200 import _lib

    L = _lib.load()
    assert L.tf_eval.argtypes[2] is ctypes.c_void_p
    assert L.tf_eval.restype is ctypes.c_int
