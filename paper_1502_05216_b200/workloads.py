"""Shard-invariant synthetic inputs for the BASELINE.json configurations.

Every element is a pure function of (seed, global index): a splitmix64
counter hash gives independent 64-bit streams per element, so any contiguous
shard [start, start+count) -- on any GPU count, or on the CPU oracle -- sees the
same values.  The numpy generator here and the CUDA generator
``tf_generate`` in csrc/tf_generate.cu perform the same integer hashing and
the same IEEE double operations (no contraction), so their outputs are
bit-identical (tests/test_gpu_parity.py::test_generator_matches_numpy).

Distributions (BASELINE.json "configs"):
  exp64        x0 ~ U[-700, 700]                          (cfg 1, cfg 5 texp)
  pow10_64     x0 = +-s*10^-e, s~U[1,10), e~UniformInt[0,300]      (cfg 2 texpm1)
  pow10c_64    pow10_64 clamped to [-1+2^-52, 1e300]                (cfg 2 tlog1p)
  log64        x0 = 2^e*m, e~UniformInt[-1022,1023], m~U[1,2); 5% -> 1+d,
               |d| <= 2^-40                                          (cfg 3)
  exp32        x0 ~ U[-87, 88] rounded to binary32                   (cfg 4 exp family)
  log32        x0 = 2^e*m, e~UniformInt[-126,127], m~U[1,2) binary32 (cfg 4 log family)
  exp64s       exp64 plus 1% specials at hashed positions           (cfg 5 texp)
  logu64s      2^e*m, e~UniformInt[-1022,1022], m~U[1,2) (log-uniform stand-in)
               plus 1% specials                                      (cfg 5 tlog)
and everywhere x1 = (x0 * u) * 2^-p with u ~ U[-1, 1] (p = 53 / 24), x1 = 0 at
special positions.  The data is synthetic: the reference has no dataset.
"""

from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

DISTS = ("exp64", "pow10_64", "pow10c_64", "log64", "exp32", "log32", "exp64s", "logu64s")
DIST_CODE = {name: i for i, name in enumerate(DISTS)}

# BASELINE.json configs -> (function, width, dist, N)
CONFIGS = {
    "cfg1_texp_f64": ("texp", 64, "exp64", 1 << 20),
    "cfg2_texpm1_f64": ("texpm1", 64, "pow10_64", 1 << 24),
    "cfg2_tlog1p_f64": ("tlog1p", 64, "pow10c_64", 1 << 24),
    "cfg3_tlog_f64": ("tlog", 64, "log64", 1 << 26),
    "cfg4_texp_f32": ("texp", 32, "exp32", 1 << 28),
    "cfg4_texpm1_f32": ("texpm1", 32, "exp32", 1 << 28),
    "cfg4_tlog_f32": ("tlog", 32, "log32", 1 << 28),
    "cfg4_tlog1p_f32": ("tlog1p", 32, "log32", 1 << 28),
    "cfg5_texp_f64": ("texp", 64, "exp64s", 1 << 30),
    "cfg5_tlog_f64": ("tlog", 64, "logu64s", 1 << 30),
}

# 10^-e for e = 0..300, correctly rounded decimal -> binary64 conversions
POW10_NEG = np.array([float(f"1e-{e}") for e in range(301)], dtype=np.float64)

_LO64 = float.fromhex("-0x1.74385446d71c4p+9")
_HI64 = float.fromhex("0x1.62e42fefa39f0p+9")
# cfg 5 special values (SURVEY.md section 8(d) cfg 5)
SPECIALS_EXP64 = np.array([
    0.0, -0.0, math.inf, -math.inf, math.nan, 5e-324, -5e-324, 2.2250738585072009e-308,
    _LO64, math.nextafter(_LO64, -math.inf), math.nextafter(_LO64, math.inf),
    _HI64, math.nextafter(_HI64, math.inf), math.nextafter(_HI64, -math.inf),
    -745.13, -708.40, 709.78, 709.782712893384,
], dtype=np.float64)
SPECIALS_LOG64 = np.array([
    0.0, -0.0, math.inf, -math.inf, math.nan, 5e-324, -5e-324, 2.2250738585072009e-308,
    2.225073858507201e-308 / 3, 1.0, -1.0, 1.7976931348623157e308, 0.5, 2.0,
    math.nextafter(1.0, 0.0), math.nextafter(1.0, 2.0), 4.9406564584124654e-322,
    1e-320,
], dtype=np.float64)


def _mix(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> int:
    """Per-(seed, stream) 64-bit key; identical in csrc/tf_generate.cu."""
    z = np.array([(seed * GOLDEN + stream * 0xD1B54A32D192ED03) & M64], dtype=np.uint64)
    return int(_mix(z)[0])


def hash_u64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    key = np.uint64(stream_key(seed, stream))
    with np.errstate(over="ignore"):
        z = key + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(GOLDEN)
        return _mix(z)


def u01(h: np.ndarray) -> np.ndarray:
    """[0, 1) double from the top 53 bits (exact)."""
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def generate(dist: str, start: int, count: int, seed: int = 0):
    """(x0, x1) for global indices [start, start+count) of distribution `dist`."""
    if dist not in DIST_CODE:
        raise ValueError(f"unknown distribution {dist!r}")
    idx = np.arange(start, start + count, dtype=np.uint64)
    h0, h1, h2, h3 = (hash_u64(seed, s, idx) for s in range(4))
    v = 2.0 * u01(h1) - 1.0            # U[-1, 1) for x1
    with np.errstate(all="ignore"):
        if dist in ("exp64", "exp64s"):
            x0 = -700.0 + 1400.0 * u01(h0)
        elif dist in ("pow10_64", "pow10c_64"):
            s = 1.0 + 9.0 * u01(h0)
            e = (h2 % np.uint64(301)).astype(np.int64)
            neg = (h3 & np.uint64(1)).astype(bool)
            x0 = s * POW10_NEG[e]
            x0 = np.where(neg, -x0, x0)
            if dist == "pow10c_64":
                x0 = np.minimum(np.maximum(x0, -1.0 + 2.0 ** -52), 1e300)
        elif dist in ("log64", "logu64s"):
            m = 1.0 + (h0 >> np.uint64(12)).astype(np.float64) * 2.0 ** -52
            if dist == "log64":
                e = (h2 % np.uint64(2046)).astype(np.int64) - 1022
            else:
                e = (h2 % np.uint64(2045)).astype(np.int64) - 1022
            x0 = np.ldexp(m, e.astype(np.int32))
            if dist == "log64":
                near1 = (h3 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 < 0.05
                d = (2.0 * u01(_mix(h3)) - 1.0) * 2.0 ** -40
                x0 = np.where(near1, 1.0 + d, x0)
        elif dist == "exp32":
            x0 = (-87.0 + 175.0 * u01(h0)).astype(np.float32)
        elif dist == "log32":
            m = (1.0 + (h0 >> np.uint64(41)).astype(np.float64) * 2.0 ** -23)
            e = (h2 % np.uint64(254)).astype(np.int64) - 126
            x0 = np.ldexp(m, e.astype(np.int32)).astype(np.float32)
        if dist in ("exp32", "log32"):
            x1 = ((x0.astype(np.float64) * v) * 2.0 ** -24).astype(np.float32)
            return x0, x1
        x1 = (x0 * v) * 2.0 ** -53
        if dist in ("exp64s", "logu64s"):
            table = SPECIALS_EXP64 if dist == "exp64s" else SPECIALS_LOG64
            hs = _mix(h3 ^ np.uint64(0x5555555555555555))
            is_sp = (hs >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 < 0.01
            pick = (hs % np.uint64(table.size)).astype(np.int64)
            x0 = np.where(is_sp, table[pick], x0)
            x1 = np.where(is_sp, 0.0, x1)
    return x0, x1
