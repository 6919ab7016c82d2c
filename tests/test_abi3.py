"""Host logic of the 3D extension, no GPU: the product's exact
orient3d (FP filter + expansion) against exact rationals, its host Step 2
(cudapre3_polyhedron) against the oracle's facets, the shard merge, the
struct layout, and the 3D generators' determinism."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

import oracle
import paper_1405_3454_b200 as cp
import synth
from tests.test_oracle3_pins import _quads, orient3d_frac


def test_struct_sizes_match_the_header_layout():
    # Extremes3T: 16 + 48*8 + 48*8 + 48*12 + 64 + 64 + 8; Polyhedron3T: 16 + 384 + 64*24 + 64*36 + 16 + 32
    assert ctypes.sizeof(cp.Extremes3T) == 16 + 384 + 384 + 576 + 128 + 8
    assert ctypes.sizeof(cp.Polyhedron3T) == 16 + 384 + 1536 + 2304 + 16 + 32


def test_orient3d_exact_vs_fractions():
    rng = np.random.default_rng(77)
    zeros = 0
    for a, b, c, d in _quads(rng, 4000):
        want = orient3d_frac(a, b, c, d)
        zeros += want == 0
        assert cp.orient3d(a, b, c, d) == want, (a, b, c, d)
        assert cp.orient3d(a, c, b, d) == -want
    assert zeros > 50


def test_orient3d_filter_boundary_cases():
    """Cases the binary64 filter cannot decide go through the expansion:
    exact zeros far from the origin, huge and tiny magnitudes."""
    big, tiny = np.float32(3e38), np.float32(2 ** -149)
    o = np.zeros(3, np.float32)
    cases = [
        (o, [big, 0, 0], [0, big, 0], [0, 0, big]),
        (o, [tiny, 0, 0], [0, tiny, 0], [0, 0, tiny]),
        ([-big, tiny, 1], [big, -big, tiny], [tiny, big, -big], [1, tiny, big]),
    ]
    a = np.full(3, 2 ** 20, np.float32)
    for k in range(200):   # points exactly on / next to the plane x + y + z = 3 * 2^20 + ...
        e = np.float32(2 ** -3) * (k % 5 - 2)
        cases.append((a, a + np.float32([1, 0, 0]), a + np.float32([0, 1, 0]), a + np.float32([e, e, 0])))
    for q in cases:
        assert cp.orient3d(*q) == orient3d_frac(*q)


def _ext3_from_oracle(xyz, angles):
    """A cudapre3_extremes_t filled from the oracle's Step 1 (host only)."""
    idx, key = oracle.extremes3(xyz, angles, with_keys=True)
    c, s = oracle.coeffs(angles)
    r = cp.Extremes3T()
    r.nang = len(c)
    r.n = len(xyz)
    for j in range(cp.MAX_SLOTS3):
        r.idx[j] = -1
    for j, (i, k) in enumerate(zip(idx, key)):
        r.idx[j] = int(i)
        r.key[j] = float(k)
        r.pt[j] = cp.Pt3(*[float(v) for v in xyz[i]])
    for k in range(len(c)):
        r.c[k], r.s[k] = c[k], s[k]
    return cp.Extremes3(r)


@pytest.mark.parametrize("family", ["cube", "ball", "sphere"])
@pytest.mark.parametrize("angles", ["A", "AT", "C", "D"])
def test_host_polyhedron_matches_oracle_facets(family, angles):
    xyz = synth.generate3(family, 20_000, seed=3)
    ext = _ext3_from_oracle(xyz, angles)
    poly = cp.polyhedron3(ext)
    E = oracle.distinct3(xyz, ext.idx)
    assert poly.eidx.tolist() == E.tolist()
    assert poly.facets.tolist() == oracle.facets3(xyz, E).tolist()
    assert poly.nf >= 4
    assert poly.raw.cells == 1
    assert poly.raw.n_entries >= poly.nf       # every facet meets some cell
    assert 1 <= poly.raw.max_candidates <= poly.nf


def test_host_polyhedron_degenerate_and_ties():
    flat = np.c_[synth.generate("disk", 3000, seed=2), np.zeros(3000)].astype(np.float32)
    poly = cp.polyhedron3(_ext3_from_oracle(flat, "A"))
    assert poly.degenerate and poly.nf == 0
    lattice = np.random.default_rng(1).integers(-2, 3, (5000, 3)).astype(np.float32)   # coplanar faces, ties
    ext = _ext3_from_oracle(lattice, "A")
    poly = cp.polyhedron3(ext)
    E = oracle.distinct3(lattice, ext.idx)
    assert poly.facets.tolist() == oracle.facets3(lattice, E).tolist()


def test_merge3_equals_unsharded_oracle():
    xyz = np.round(synth.generate3("ball", 30_001, seed=4) * 16).astype(np.float32)   # heavy ties
    whole = oracle.extremes3(xyz, "A")
    parts = []
    bounds = [0, 7_000, 7_001, 19_000, 30_001]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        e = _ext3_from_oracle(xyz[lo:hi], "A")
        for j in range(24):
            e.raw.idx[j] += lo
        parts.append(e)
    m = cp.merge3(parts)
    assert m.idx.tolist() == whole.tolist()
    assert m.n == len(xyz)


def test_generate3_is_deterministic_and_sliceable():
    a = synth.generate3("sphere", 5000, seed=9)
    b = synth.generate3("sphere", 2000, seed=9, base=3000)
    assert np.array_equal(a[3000:], b)
    r = np.sqrt((a.astype(np.float64) ** 2).sum(1))
    assert (r <= 1.0 + 1e-6).all() and (r >= 1 - 1e-3 - 1e-6).all()
    c = synth.generate3("ball", 5000, seed=9)
    assert ((c.astype(np.float64) ** 2).sum(1) <= 1.0 + 1e-6).all()


def _exit_facets(fv, o, d):
    """Facets through which rays o + t d (rows of d) leave the polyhedron, by
    binary64 ray casting: per ray the set achieving the smallest exit t
    (ties: the ray passes through an edge or vertex)."""
    a, b, c = (fv[:, k, :].astype(np.float64) for k in range(3))
    n = np.cross(b - a, c - a)                       # inward normals (E on the positive side)
    oo = np.einsum("fk,fk->f", n, o[None, :] - a)    # orient(o) > 0: o strictly inside
    nd = d @ n.T                                     # N . d
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.where(nd < 0, oo[None, :] / -nd, np.inf)
    tmin = t.min(axis=1, keepdims=True)
    return t <= tmin * (1 + 1e-9) + 1e-300


@pytest.mark.parametrize("family", ["ball", "cube", "sphere"])
@pytest.mark.parametrize("angles", ["A", "D"])
def test_direction_cells_contain_the_exit_facet(family, angles):
    """The argument behind K2-3D: a point is strictly inside
    iff it is strictly inside the facet its ray from the centre leaves
    through, so every direction cell's candidate list must contain that exit
    facet — for random directions and for directions on both sides of every
    cell boundary (where the kernel's rounded cell index may land next door,
    covered by the guard)."""
    xyz = synth.generate3(family, 50_000, seed=11)
    ext = _ext3_from_oracle(xyz, angles)
    poly = cp.polyhedron3(ext)
    masks, centre, G, used = cp.cells3(ext)
    assert used and poly.nf >= 4
    fv = np.frombuffer(bytes(poly.raw.fv), np.float32).reshape(-1, 3, 3)[: poly.nf]
    o = centre.astype(np.float64)
    rng = np.random.default_rng(5)
    d = rng.normal(size=(60_000, 3))
    # directions just off the cell boundaries: u, v on the grid lines +- 1e-7
    face_axis = rng.integers(0, 3, 20_000)
    sign = rng.choice([-1.0, 1.0], 20_000)
    grid = -1.0 + 2.0 * rng.integers(0, G + 1, (20_000, 2)) / G
    uv = grid + rng.choice([-1e-7, 1e-7], (20_000, 2)) + rng.uniform(-1, 1, (20_000, 2)) * [[0, 1]] * 0.5
    uv = np.clip(uv, -1.0, 1.0)
    e = np.zeros((20_000, 3))
    U, V = np.array([1, 2, 0]), np.array([2, 0, 1])
    e[np.arange(20_000), face_axis] = sign
    e[np.arange(20_000), U[face_axis]] = uv[:, 0]
    e[np.arange(20_000), V[face_axis]] = uv[:, 1]
    d = np.concatenate([d, e])
    ex = _exit_facets(fv, o, d)
    # the cell of each direction, exactly as defined (binary64 division)
    ad = np.abs(d)
    axis = np.where((ad[:, 0] >= ad[:, 1]) & (ad[:, 0] >= ad[:, 2]), 0, np.where(ad[:, 1] >= ad[:, 2], 1, 2))
    m = d[np.arange(len(d)), axis]
    u = d[np.arange(len(d)), U[axis]] / np.abs(m)
    v = d[np.arange(len(d)), V[axis]] / np.abs(m)
    # the exact cell, and the cells the kernel's rounded (u, v) (error < 2^-20)
    # may land in: perturbations of 2^-18 must be covered by the 2^-12 guard
    for du, dv in ((0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)):
        uu, vv = u + du * 2.0 ** -18, v + dv * 2.0 ** -18
        iu = np.clip(np.floor((uu + 1) * G / 2), 0, G - 1).astype(int)
        iv = np.clip(np.floor((vv + 1) * G / 2), 0, G - 1).astype(int)
        cell = ((2 * axis + (m < 0)) * G + iu) * G + iv
        bits = (masks[cell][:, None] >> np.arange(poly.nf, dtype=np.uint64)[None, :]) & np.uint64(1)
        covered = (ex & bits.astype(bool)).any(axis=1)
        assert covered.all(), f"{(~covered).sum()} of {len(d)} directions miss their exit facet ({du}, {dv})"


def _fma32(a, b, c):
    """RN32(a*b + c) for float32 arrays: a*b is exact in binary64 and the
    float64 sum is within 2^-53 relative, far below the float32 rounding."""
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


@pytest.mark.parametrize("family,scale,offset", [("ball", 1.0, 0.0), ("cube", 1.0, 0.0),
                                                 ("ball", 1e3, 5e3), ("cube", 1e-3, 0.0)])
def test_plane_test_error_bound(family, scale, offset):
    """The bound K2-3D's fast decisions rest on: over the data
    bounding box, |float plane test - orient3d| <= E for every facet —
    checked on random points, the box corners and the points themselves, with
    orient3d evaluated in binary64 (its own error ~2^-50 S is far below E)."""
    xyz = ((synth.generate3(family, 30_000, seed=13).astype(np.float64) * scale) + offset).astype(np.float32)
    ext = _ext3_from_oracle(xyz, "A")
    poly = cp.polyhedron3(ext)
    pl = cp.planes3(ext)
    assert len(pl) == poly.nf >= 4 and np.isfinite(pl[:, 4]).all()
    fv = np.frombuffer(bytes(poly.raw.fv), np.float32).reshape(-1, 3, 3)[: poly.nf].astype(np.float64)
    lo, hi = xyz.min(0), xyz.max(0)
    rng = np.random.default_rng(2)
    corners = np.array([[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1]) for z in (lo[2], hi[2])],
                       np.float32)
    pts = np.concatenate([rng.uniform(lo, hi, (20_000, 3)).astype(np.float32), corners, xyz[:5000]])
    for f in range(poly.nf):
        A, B, C, D, E = pl[f]
        g = _fma32(np.full(len(pts), A, np.float32), pts[:, 0],
                   _fma32(np.full(len(pts), B, np.float32), pts[:, 1],
                          _fma32(np.full(len(pts), C, np.float32), pts[:, 2], np.full(len(pts), D, np.float32))))
        a, b, c = fv[f]
        exact = (pts.astype(np.float64) - a) @ np.cross(b - a, c - a)
        err = np.abs(g.astype(np.float64) - exact)
        assert (err <= E).all(), (f, float(err.max()), float(E))
        assert float(err.max()) > 0 or E > 0
