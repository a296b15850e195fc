"""ctypes binding of libtwofold_b200.so (the C ABI declared in include/twofold_b200.h).

The product path has no fallback: if the library is missing, or no CUDA device
is visible, every compute call raises RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TWOFOLD_B200_LIB") or os.path.join(HERE, "lib", "libtwofold_b200.so")
CSRC = os.path.join(HERE, "csrc")

TF_OK, TF_ERR_ARG, TF_ERR_CUDA = 0, -1, -2
# tf_eval function codes (include/twofold_b200.h TF_FN_*)
FN_CODES = {"texp": 0, "texpm1": 1, "tlog": 2, "tlog1p": 3, "pexp0": 4, "texp0": 5, "texpp": 6,
            "pexp": 7, "pexpm10": 8, "texpm10": 9, "texpm1p": 10, "pexpm1": 11, "plog0": 12,
            "tlog0": 13, "tlogp": 14, "plog": 15, "plog1p0": 16, "tlog1p0": 17, "tlog1pp": 18,
            "plog1p": 19}
FLAG_FORCE_EXACT = 1
FLAG_COUNT_EXACT = 2
FLAG_MARK_EXACT = 4
DIST_CODES = {"exp64": 0, "pow10_64": 1, "pow10c_64": 2, "log64": 3, "exp32": 4, "log32": 5,
              "exp64s": 6, "logu64s": 7}

# every symbol include/twofold_b200.h declares (checked by tests/test_abi.py)
EXPORTS = ("tf_version", "tf_last_error", "tf_init", "tf_texp_f64", "tf_texpm1_f64",
           "tf_tlog_f64", "tf_tlog1p_f64", "tf_texp_f32", "tf_texpm1_f32", "tf_tlog_f32",
           "tf_tlog1p_f32", "tf_eval", "tf_generate", "tf_compare", "tf_fma_peak",
           "tf_exact_count", "tf_audit_errors", "tf_etalon", "tf_checksum", "tf_eft",
           "tf_eval_host", "tf_reduce_stats")
# tf_eft op codes (include/twofold_b200.h TF_OP_*)
OP_CODES = {"fast_two_sum": 0, "two_sum": 1, "two_diff": 2, "two_prod": 3, "split": 4,
            "renorm_fast": 5, "renorm": 6, "t_add": 7, "t_add_d": 8, "t_mul": 9, "t_mul_d": 10,
            "t_div": 11, "t_sqrt": 12}
FAMILY_CODES = {"exp": 0, "expm1": 1, "log": 2, "log1p": 3}
ETALON_CODES = {"oracle": 0, "lib": 1}
AUDIT_INCLUDED, AUDIT_FLOOR, AUDIT_DOMAIN, AUDIT_ABSOLUTE = 0, 1, 2, 3



class TfStats(ctypes.Structure):
    """struct tf_stats (include/twofold_b200.h): one shard's parity / error statistics."""

    _fields_ = [("n", ctypes.c_uint64), ("z0_mismatch", ctypes.c_uint64),
                ("z0_gt1ulp", ctypes.c_uint64), ("tol_violations", ctypes.c_uint64),
                ("class_mismatch", ctypes.c_uint64), ("z1_mismatch", ctypes.c_uint64),
                ("included", ctypes.c_uint64), ("warnings", ctypes.c_uint64),
                ("err_sum", ctypes.c_double), ("err_max", ctypes.c_double)]


STATS_COUNT_KEYS = ("n", "z0_mismatch", "z0_gt1ulp", "tol_violations", "class_mismatch",
                    "z1_mismatch", "included", "warnings")


_lib = None
_lock = threading.Lock()
_inited: set[int] = set()


def build(force: bool = False) -> str:
    """Compile the CUDA library in-tree for sm_100a (nvcc; see csrc/Makefile)."""
    args = ["make", "-s", f"-j{min(4, os.cpu_count() or 1)}", "-C", CSRC]
    if force:
        args.insert(1, "-B")
    subprocess.run(args, check=True)
    return LIB_PATH


def load() -> ctypes.CDLL:
    """Load the shared library (no CUDA context is created here)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libtwofold_b200.so not found at {LIB_PATH}; run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (or make -C "
                f"{CSRC}) first -- there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.tf_version.restype = i32
        L.tf_last_error.restype = ctypes.c_char_p
        L.tf_init.argtypes = [i32]
        L.tf_init.restype = i32
        for fn in ("texp", "texpm1", "tlog", "tlog1p"):
            for w in ("f64", "f32"):
                f = getattr(L, f"tf_{fn}_{w}")
                f.argtypes = [vp, vp, vp, vp, i64, vp]
                f.restype = i32
        L.tf_eval.argtypes = [i32, i32, vp, vp, vp, vp, i64, vp, i32]
        L.tf_eval.restype = i32
        L.tf_generate.argtypes = [i32, ctypes.c_uint64, i64, i64, vp, vp, vp]
        L.tf_generate.restype = i32
        L.tf_compare.argtypes = [i32, vp, vp, vp, vp, i64, ctypes.c_double, ctypes.c_double,
                                 vp, vp]
        L.tf_compare.restype = i32
        L.tf_fma_peak.argtypes = [i32, vp, i32, i32, vp]
        L.tf_fma_peak.restype = i32
        L.tf_exact_count.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), i32]
        L.tf_exact_count.restype = i32
        L.tf_audit_errors.argtypes = [i32, i32, i32, vp, vp, vp, vp, i64, vp, vp, vp]
        L.tf_audit_errors.restype = i32
        L.tf_etalon.argtypes = [i32, vp, vp, i64, vp, vp, vp]
        L.tf_etalon.restype = i32
        L.tf_checksum.argtypes = [i32, vp, i64, vp, vp]
        L.tf_checksum.restype = i32
        L.tf_eft.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, vp, i64, vp]
        L.tf_eft.restype = i32
        L.tf_eval_host.argtypes = [i32, i32, vp, vp, vp, vp, i64, i64, vp, i32]
        L.tf_eval_host.restype = i32
        if hasattr(L, "tf_reduce_stats"):      # (older diagnostic builds lack it)
            L.tf_reduce_stats.argtypes = [ctypes.POINTER(TfStats), i64, ctypes.POINTER(TfStats)]
            L.tf_reduce_stats.restype = i32
        _lib = L
        return L


def reduce_stats_c(parts: list[TfStats]) -> TfStats:
    """Merge shard statistics with the C ABI's tf_reduce_stats (host code only:
    works without a GPU)."""
    L = load()
    arr = (TfStats * max(1, len(parts)))(*parts)
    out = TfStats()
    check(L.tf_reduce_stats(arr, len(parts), ctypes.byref(out)), "tf_reduce_stats")
    return out


def check(rc: int, what: str) -> None:
    if rc != TF_OK:
        msg = load().tf_last_error().decode(errors="replace")
        if rc == TF_ERR_ARG:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what}: {msg}")


_scalar_dev = None


def scalar_device() -> ctypes.CDLL:
    """The library, initialised on torch's current device (scalar-call fast path:
    checked once per process and device)."""
    global _scalar_dev
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the twofold kernels need a B200 "
                           "(sm_100a); there is no CPU fallback")
    d = torch.cuda.current_device()
    if _scalar_dev != d:
        ensure_device(d)
        _scalar_dev = d
    return _lib


def ensure_device(device_index: int) -> ctypes.CDLL:
    L = load()
    if device_index not in _inited:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device visible: the twofold kernels need a B200 "
                               "(sm_100a); there is no CPU fallback")
        with torch.cuda.device(device_index):
            check(L.tf_init(-1), "tf_init")
        _inited.add(device_index)
    return L
