"""CPU oracle for the CudaPre filter (arXiv 1405.3454) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_1405_3454_b200``) never imports it and shares no code with it.

The arithmetic lives in ``cudapre_oracle.c`` (plain C, binary64, compiled with
``-ffp-contract=off -fno-fast-math``); this module only compiles it with gcc,
loads it with ctypes and marshals numpy arrays.  Every function cites the
passage of PAPER.md (P:nn) / SPEC.md (S:nn) it follows; see the C file header.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cudapre_oracle.c")
_SRC3 = os.path.join(_HERE, "cudapre3_oracle.c")   # the 3D extension
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (idempotent)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_SRC3))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, _SRC3, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, f32, f64, i32 = ctypes.c_int64, ctypes.c_float, ctypes.c_double, ctypes.c_int
        vp = ctypes.c_void_p
        lib.oracle_coeffs.argtypes = [f64, ctypes.POINTER(f64), ctypes.POINTER(f64)]
        lib.oracle_coeffs.restype = i32
        lib.oracle_orient.argtypes = [f32] * 6
        lib.oracle_orient.restype = i32
        lib.oracle_extremes.argtypes = [vp, i64, vp, vp, i32, i32, vp, vp]
        lib.oracle_extremes.restype = i32
        lib.oracle_hull.argtypes = [vp, vp, i64, vp]
        lib.oracle_hull.restype = i64
        lib.oracle_strictly_inside.argtypes = [vp, i64, f32, f32]
        lib.oracle_strictly_inside.restype = i32
        lib.oracle_filter_mask.argtypes = [vp, i64, vp, i64, i32, vp]
        lib.oracle_filter_mask.restype = None
        lib.oracle_cudapre.argtypes = [vp, i64, vp, vp, i32, i32, vp, vp, vp, vp]
        lib.oracle_cudapre.restype = i32
        lib.oracle3_orient.argtypes = [vp, vp, vp, vp]
        lib.oracle3_orient.restype = i32
        lib.oracle3_extremes.argtypes = [vp, i64, vp, vp, i32, i32, vp, vp]
        lib.oracle3_extremes.restype = i32
        lib.oracle3_distinct.argtypes = [vp, vp, i64, vp]
        lib.oracle3_distinct.restype = i64
        lib.oracle3_facets.argtypes = [vp, vp, i64, vp, i64]
        lib.oracle3_facets.restype = i64
        lib.oracle3_strictly_inside.argtypes = [vp, i64, vp]
        lib.oracle3_strictly_inside.restype = i32
        lib.oracle3_filter_mask.argtypes = [vp, i64, vp, i64, i32, vp]
        lib.oracle3_filter_mask.restype = None
        lib.oracle3_cudapre.argtypes = [vp, i64, vp, vp, i32, i32, vp, vp, i64, vp, vp]
        lib.oracle3_cudapre.restype = i32
        _lib = lib
    return _lib


def _pts(xy) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(xy, dtype=np.float32).reshape(-1, 2))
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


PRESETS = {"A": (0.0, 30.0, 45.0, 60.0), "B": (0.0, 30.0, 45.0, 45.0), "AT": (0.0,),
           "C": (0.0, 22.5, 45.0, 67.5), "D": (0.0, 15.0, 22.5, 30.0, 45.0, 60.0, 67.5, 75.0)}


def coeffs(angles) -> tuple[np.ndarray, np.ndarray]:
    """Correctly rounded (cos, sin) of each angle in degrees (reading A5)."""
    lib = _load()
    if isinstance(angles, str):
        angles = PRESETS[angles]
    c = np.empty(len(angles), np.float64)
    s = np.empty(len(angles), np.float64)
    for k, a in enumerate(angles):
        cc, ss = ctypes.c_double(), ctypes.c_double()
        if lib.oracle_coeffs(float(a), ctypes.byref(cc), ctypes.byref(ss)) != 0:
            raise ValueError(f"oracle has no correctly rounded coefficients for {a} deg")
        c[k], s[k] = cc.value, ss.value
    return c, s


def orient(a, b, c) -> int:
    """Exact sign of (b-a) x (c-a) for float inputs (reading A11)."""
    return int(_load().oracle_orient(float(a[0]), float(a[1]), float(b[0]), float(b[1]),
                                     float(c[0]), float(c[1])))


def extremes(xy, angles="A", threads: int = 1, with_keys: bool = False):
    """Step 1: the 4*len(angles) extreme-point indices.

    Slot 4k+{0,1,2,3} = argmin X_k, argmax X_k, argmin Y_k, argmax Y_k with
    X_k = RN(RN(x c_k)+RN(y s_k)), Y_k = RN(RN(y c_k)-RN(x s_k)), lowest index
    on ties.  Raises ValueError on empty input."""
    p = _pts(xy)
    c, s = coeffs(angles)
    idx = np.empty(4 * len(c), np.int64)
    key = np.empty(4 * len(c), np.float64)
    rc = _load().oracle_extremes(_ptr(p), len(p), _ptr(c), _ptr(s), len(c), threads,
                                 _ptr(idx), _ptr(key))
    if rc != 0:
        raise ValueError("empty input")
    return (idx, key) if with_keys else idx


def hull(xy, ids=None) -> np.ndarray:
    """Andrew's monotone chain: canonical CCW ring of
    vertex ids starting at the lexicographically smallest vertex; collinear
    points excluded; duplicates represented by their lowest id.  Length 1 or
    2 means a degenerate point / segment."""
    p = _pts(xy)
    if ids is None:
        m = len(p)
        ids_a = None
    else:
        ids_a = np.ascontiguousarray(np.asarray(ids, dtype=np.int64))
        m = len(ids_a)
    ring = np.empty(max(m, 1), np.int64)
    k = _load().oracle_hull(_ptr(p), None if ids_a is None else _ptr(ids_a), m, _ptr(ring))
    if k < 0:
        raise MemoryError
    return ring[:k].copy()


def polygon(xy, ext_idx) -> np.ndarray:
    """Step 2: ring of the distinct extreme candidates."""
    return hull(xy, np.asarray(ext_idx, np.int64))


def strictly_inside(ring_xy, p) -> bool:
    r = _pts(ring_xy)
    return bool(_load().oracle_strictly_inside(_ptr(r), len(r), float(p[0]), float(p[1])))


def filter_mask(xy, ring_xy, threads: int = 1) -> np.ndarray:
    """Step 3: keep[i] = not strictly inside the ring."""
    p = _pts(xy)
    r = _pts(ring_xy)
    keep = np.zeros(len(p), np.uint8)
    _load().oracle_filter_mask(_ptr(p), len(p), _ptr(r), len(r), threads, _ptr(keep))
    return keep.astype(bool)


def cudapre(xy, angles="A", threads: int = 1) -> dict:
    """The whole method in the paper's order: returns a dict with
    ``ext_idx`` (Step 1), ``ring`` (Step 2 vertex ids), ``degenerate``,
    ``survivors`` (Step 3, ascending int64 indices)."""
    p = _pts(xy)
    if len(p) == 0:
        raise ValueError("empty input")
    c, s = coeffs(angles)
    ext = np.empty(4 * len(c), np.int64)
    ring = np.empty(4 * len(c), np.int64)
    nv = np.zeros(1, np.int64)
    keep = np.zeros(len(p), np.uint8)
    rc = _load().oracle_cudapre(_ptr(p), len(p), _ptr(c), _ptr(s), len(c), threads,
                                _ptr(ext), _ptr(ring), _ptr(nv), _ptr(keep))
    if rc != 0:
        raise ValueError("empty input")
    nvv = int(nv[0])
    return {
        "ext_idx": ext,
        "ring": ring[:nvv].copy(),
        "degenerate": nvv < 3,
        "survivors": np.flatnonzero(keep).astype(np.int64),
    }


# ---------------------------------------------------------------------------
# The 3D extension (readings B1-B6 in DESIGN.md §3).
# The arithmetic lives in cudapre3_oracle.c.

MAX_FACETS3 = 4096


def _pts3(xyz) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(xyz, dtype=np.float32).reshape(-1, 3))


def orient3d(a, b, c, d) -> int:
    """Exact sign of det[b-a; c-a; d-a] for float inputs (reading B6)."""
    q = [np.ascontiguousarray(np.asarray(v, np.float32).reshape(3)) for v in (a, b, c, d)]
    return int(_load().oracle3_orient(*[_ptr(v) for v in q]))


def extremes3(xyz, angles="A", threads: int = 1, with_keys: bool = False):
    """Step 1 in 3D (P:115 with P:33-35; B1, B2): 6*len(angles) indices, slot
    6k+{minX, maxX, minY, maxY, minZ, maxZ} of the frame rotated by angle k
    about z; lowest index on ties.  Raises ValueError on empty input."""
    p = _pts3(xyz)
    c, s = coeffs(angles)
    idx = np.empty(6 * len(c), np.int64)
    key = np.empty(6 * len(c), np.float64)
    if _load().oracle3_extremes(_ptr(p), len(p), _ptr(c), _ptr(s), len(c), threads, _ptr(idx),
                                _ptr(key)) != 0:
        raise ValueError("empty input")
    return (idx, key) if with_keys else idx


def distinct3(xyz, picks) -> np.ndarray:
    """E: the distinct picks, ascending index, equal coordinates -> lowest index (B3)."""
    p = _pts3(xyz)
    pk = np.ascontiguousarray(np.asarray(picks, np.int64))
    E = np.empty(max(len(pk), 1), np.int64)
    m = _load().oracle3_distinct(_ptr(p), _ptr(pk), len(pk), _ptr(E))
    if m < 0:
        raise ValueError("too many picks")
    return E[:m].copy()


def facets3(xyz, E) -> np.ndarray:
    """Step 2 in 3D (B3, B4): (nf, 3) point ids of the first supporting triple
    of each facet plane of conv(E), E on the positive side; nf = 0 means
    degenerate (|E| < 4 or coplanar)."""
    p = _pts3(xyz)
    Ea = np.ascontiguousarray(np.asarray(E, np.int64))
    out = np.empty((MAX_FACETS3, 3), np.int64)
    nf = _load().oracle3_facets(_ptr(p), _ptr(Ea), len(Ea), _ptr(out), MAX_FACETS3)
    if nf < 0:
        raise ValueError("facet overflow")
    return out[:nf].copy()


def strictly_inside3(fxyz, p) -> bool:
    """1 iff orient3d(f, p) > 0 for every facet (fxyz: (nf, 3, 3) coordinates)."""
    f = np.ascontiguousarray(np.asarray(fxyz, np.float32).reshape(-1, 9))
    q = np.ascontiguousarray(np.asarray(p, np.float32).reshape(3))
    return bool(_load().oracle3_strictly_inside(_ptr(f), len(f), _ptr(q)))


def filter_mask3(xyz, fxyz, threads: int = 1) -> np.ndarray:
    """Step 3 in 3D (B5): keep[i] = not strictly inside the polyhedron."""
    p = _pts3(xyz)
    f = np.ascontiguousarray(np.asarray(fxyz, np.float32).reshape(-1, 9))
    keep = np.zeros(len(p), np.uint8)
    _load().oracle3_filter_mask(_ptr(p), len(p), _ptr(f), len(f), threads, _ptr(keep))
    return keep.astype(bool)


def cudapre3(xyz, angles="A", threads: int = 1) -> dict:
    """The 3D method in order: ``ext_idx`` (Step 1), ``facets`` (Step 2,
    (nf, 3) ids), ``degenerate``, ``survivors`` (Step 3, ascending int64)."""
    p = _pts3(xyz)
    if len(p) == 0:
        raise ValueError("empty input")
    c, s = coeffs(angles)
    ext = np.empty(6 * len(c), np.int64)
    fac = np.empty((MAX_FACETS3, 3), np.int64)
    nf = np.zeros(1, np.int64)
    keep = np.zeros(len(p), np.uint8)
    if _load().oracle3_cudapre(_ptr(p), len(p), _ptr(c), _ptr(s), len(c), threads, _ptr(ext),
                               _ptr(fac), MAX_FACETS3, _ptr(nf), _ptr(keep)) != 0:
        raise ValueError("empty input")
    k = int(nf[0])
    return {
        "ext_idx": ext,
        "facets": fac[:k].copy(),
        "degenerate": k == 0,
        "survivors": np.flatnonzero(keep).astype(np.int64),
    }
