"""Seeded synthetic point generators (input recipe).

This module is the ONE thing the oracle side and the CUDA side share: it
produces input bytes and holds none of the method's arithmetic.  It has two
bit-identical implementations of the same counter-based generator:

* ``generate(...)`` here — numpy, host side (used by the oracle tests);
* ``synth/gen.cu`` → ``libsynth.so`` — a CUDA kernel that writes the same
  bytes straight into HBM (used by bench.py and the GPU tests for sizes the
  host would take minutes to produce).  ``synth.cuda.generate`` wraps it.

Every output value is a fixed sequence of IEEE round-to-nearest operations on
float32/float64 with no fused multiply-add and no library transcendental, so
both implementations agree bit for bit (checked in tests/test_gpu_parity.py).

Counter-based RNG: SplitMix64 finaliser of
``key(seed) + (((i << 7) | (attempt << 1) | stream) + 1) * GOLDEN``; each draw
gives two 24-bit uniforms ``u = k * 2**-24`` (exact floats).  Point i depends
only on (seed, i), so any index range [base, base+n) can be generated alone
(shards, samples).

Families (paper §3):
  square  uniform in [lo, hi)^2                 x = RN(RN(u*w) + lo), w = RN(hi-lo)
  disk    uniform in the unit disk              per-index rejection from [-1,1)^2, x^2+y^2 <= 1 (float32)
  gauss   N(0,1)^2 (Marsaglia polar method)     f = sqrt(-2 ln s / s) with an RN-only log series
  circle  near-circle r in [1-eps, 1], uniform angle (direction of a disk sample, radius 1-eps*u3)
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
SEED_SALT = np.uint64(0x632BE59BD9B4E019)
MAX_ATTEMPTS = 64
INV24 = np.float32(2.0 ** -24)

# RN-only natural log (gauss family): ln s = e*LN2 + 2 t (1 + t^2/3 + ... + t^18/19),
# t = (m-1)/(m+1), m in [sqrt(1/2), sqrt(2)).  Coefficients as exact hex literals,
# shared verbatim with synth/gen.cu.
LN2 = float.fromhex("0x1.62e42fefa39efp-1")
SQRT_HALF = float.fromhex("0x1.6a09e667f3bcdp-1")
LOG_COEF = [float.fromhex(h) for h in (
    "0x1.0000000000000p+0",   # 1
    "0x1.5555555555555p-2",   # 1/3
    "0x1.999999999999ap-3",   # 1/5
    "0x1.2492492492492p-3",   # 1/7
    "0x1.c71c71c71c71cp-4",   # 1/9
    "0x1.745d1745d1746p-4",   # 1/11
    "0x1.3b13b13b13b14p-4",   # 1/13
    "0x1.1111111111111p-4",   # 1/15
    "0x1.e1e1e1e1e1e1ep-5",   # 1/17
    "0x1.af286bca1af28p-5",   # 1/19
)]

FAMILIES = ("square", "disk", "gauss", "circle")


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * M1
    z = z ^ (z >> np.uint64(27))
    z = z * M2
    return z ^ (z >> np.uint64(31))


def seed_key(seed: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return _mix64(np.asarray([np.uint64(seed) * GOLDEN + SEED_SALT], np.uint64))[0]


def draw(key: np.uint64, idx: np.ndarray, attempt: int, stream: int) -> np.ndarray:
    ctr = (idx.astype(np.uint64) << np.uint64(7)) | np.uint64((attempt << 1) | stream)
    with np.errstate(over="ignore"):
        return _mix64(key + (ctr + np.uint64(1)) * GOLDEN)


def _uniforms(z: np.ndarray):
    u1 = (z >> np.uint64(40)).astype(np.float32) * INV24
    u2 = ((z >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.float32) * INV24
    return u1, u2


def _ln(s: np.ndarray) -> np.ndarray:
    """RN-only natural log of positive float64 values (generator use only)."""
    m, e = np.frexp(s)                     # s = m 2^e, m in [0.5, 1)
    lo = m < SQRT_HALF
    m = np.where(lo, m * 2.0, m)
    e = np.where(lo, e - 1, e).astype(np.float64)
    t = (m - 1.0) / (m + 1.0)
    t2 = t * t
    p = np.full_like(t, LOG_COEF[-1])
    for cf in reversed(LOG_COEF[:-1]):
        p = p * t2
        p = p + cf
    lm = t * p
    lm = lm * 2.0
    return e * LN2 + lm


def _pm1(u: np.ndarray) -> np.ndarray:
    """2u - 1 in float32 (exact for u = k 2^-24)."""
    return u * np.float32(2.0) - np.float32(1.0)


def _gen_chunk(family: str, key, idx: np.ndarray, lo: float, hi: float, eps: float) -> np.ndarray:
    n = len(idx)
    out = np.zeros((n, 2), np.float32)
    if family == "square":
        u1, u2 = _uniforms(draw(key, idx, 0, 0))
        w = np.float32(hi) - np.float32(lo)
        out[:, 0] = u1 * w + np.float32(lo)
        out[:, 1] = u2 * w + np.float32(lo)
        return out
    pending = np.arange(n)
    for attempt in range(MAX_ATTEMPTS):
        if len(pending) == 0:
            break
        u1, u2 = _uniforms(draw(key, idx[pending], attempt, 0))
        x = _pm1(u1)
        y = _pm1(u2)
        s = x * x + y * y                  # float32, two RN products then RN sum
        if family == "disk":
            ok = s <= np.float32(1.0)
            out[pending[ok], 0] = x[ok]
            out[pending[ok], 1] = y[ok]
        elif family == "gauss":
            ok = (s > np.float32(0.0)) & (s < np.float32(1.0))
            sd = s[ok].astype(np.float64)
            f = np.sqrt((_ln(sd) * -2.0) / sd)
            out[pending[ok], 0] = (x[ok].astype(np.float64) * f).astype(np.float32)
            out[pending[ok], 1] = (y[ok].astype(np.float64) * f).astype(np.float32)
        elif family == "circle":
            ok = (s > np.float32(0.0)) & (s <= np.float32(1.0))
            xd = x[ok].astype(np.float64)
            yd = y[ok].astype(np.float64)
            d = np.sqrt(xd * xd + yd * yd)
            u3, _ = _uniforms(draw(key, idx[pending[ok]], attempt, 1))
            r = 1.0 - eps * u3.astype(np.float64)
            sc = r / d
            out[pending[ok], 0] = (xd * sc).astype(np.float32)
            out[pending[ok], 1] = (yd * sc).astype(np.float32)
        else:
            raise ValueError(f"unknown family {family!r}")
        pending = pending[~ok]
    return out  # points that never accepted stay (0, 0); probability < 1e-40


def generate(family: str, n: int, seed: int, base: int = 0, *, lo: float = -1.0,
             hi: float = 1.0, eps: float = 1e-3, chunk: int = 1 << 22) -> np.ndarray:
    """Points [base, base+n) of the seeded stream, as a float32 (n, 2) array."""
    if family not in FAMILIES:
        raise ValueError(f"unknown family {family!r}")
    key = seed_key(seed)
    out = np.empty((n, 2), np.float32)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        idx = np.arange(base + a, base + b, dtype=np.int64)
        out[a:b] = _gen_chunk(family, key, idx, lo, hi, eps)
    return out


# ---------------------------------------------------------------------------
# 3D families (the 3D extension).  Same counter-based
# stream; a point's first draw (stream 0) gives (u1, u2), its second draw
# (stream 1) gives (u3, u4).
#   cube    uniform in [lo, hi)^3                 x = RN(RN(u*w) + lo)
#   ball    uniform in the unit ball              per-index rejection from [-1,1)^3,
#                                                 RN(RN(x^2 + y^2) + z^2) <= 1 (float32)
#   sphere  near-sphere shell r in [1-eps, 1]     direction of a ball sample, radius 1-eps*u4
FAMILIES3 = ("cube", "ball", "sphere")


def _gen3_chunk(family: str, key, idx: np.ndarray, lo: float, hi: float, eps: float) -> np.ndarray:
    n = len(idx)
    out = np.zeros((n, 3), np.float32)
    if family == "cube":
        u1, u2 = _uniforms(draw(key, idx, 0, 0))
        u3, _ = _uniforms(draw(key, idx, 0, 1))
        w = np.float32(hi) - np.float32(lo)
        for j, u in enumerate((u1, u2, u3)):
            out[:, j] = u * w + np.float32(lo)
        return out
    pending = np.arange(n)
    for attempt in range(MAX_ATTEMPTS):
        if len(pending) == 0:
            break
        u1, u2 = _uniforms(draw(key, idx[pending], attempt, 0))
        u3, u4 = _uniforms(draw(key, idx[pending], attempt, 1))
        x, y, z = _pm1(u1), _pm1(u2), _pm1(u3)
        s = (x * x + y * y) + z * z        # float32: RN products, RN sums in this order
        if family == "ball":
            ok = s <= np.float32(1.0)
            out[pending[ok]] = np.stack([x[ok], y[ok], z[ok]], 1)
        elif family == "sphere":
            ok = (s > np.float32(0.0)) & (s <= np.float32(1.0))
            xd, yd, zd = (v[ok].astype(np.float64) for v in (x, y, z))
            d = np.sqrt((xd * xd + yd * yd) + zd * zd)
            r = 1.0 - eps * u4[ok].astype(np.float64)
            sc = r / d
            out[pending[ok]] = np.stack([xd * sc, yd * sc, zd * sc], 1).astype(np.float32)
        else:
            raise ValueError(f"unknown 3D family {family!r}")
        pending = pending[~ok]
    return out


def generate3(family: str, n: int, seed: int, base: int = 0, *, lo: float = -1.0,
              hi: float = 1.0, eps: float = 1e-3, chunk: int = 1 << 22) -> np.ndarray:
    """3D points [base, base+n) of the seeded stream, as a float32 (n, 3) array."""
    if family not in FAMILIES3:
        raise ValueError(f"unknown 3D family {family!r}")
    key = seed_key(seed)
    out = np.empty((n, 3), np.float32)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        idx = np.arange(base + a, base + b, dtype=np.int64)
        out[a:b] = _gen3_chunk(family, key, idx, lo, hi, eps)
    return out


# Named configs (BASELINE.json "configs").
CONFIGS = {
    "C1": dict(family="square", n=100_000, seed=1, lo=0.0, hi=1.0),
    "C2a": dict(family="square", n=10_000_000, seed=2, lo=-1.0, hi=1.0),
    "C2b": dict(family="disk", n=10_000_000, seed=3),
    "C3": dict(family="gauss", n=50_000_000, seed=4),
    "C4": dict(family="circle", n=20_000_000, seed=5, eps=1e-3),
    "C4e0": dict(family="circle", n=20_000_000, seed=5, eps=0.0),
    "C5": dict(family="disk", n=2_000_000_000, seed=6),
}

# 3D workloads (f4; not BASELINE configs): 1e9 points = 12 GB of float3.
CONFIGS3 = {
    "T1": dict(family="ball", n=1_000_000, seed=21),
    "T3": dict(family="cube", n=1_000_000_000, seed=22),
    "T4": dict(family="ball", n=1_000_000_000, seed=23),
    "T5": dict(family="sphere", n=200_000_000, seed=24, eps=1e-3),
}


def config_kwargs(name: str) -> dict:
    cfg = dict(CONFIGS[name] if name in CONFIGS else CONFIGS3[name])
    cfg.pop("n")
    return cfg
