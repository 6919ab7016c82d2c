"""Pins for the 3D oracle (readings B1-B6 in DESIGN.md
§3).  Run with -m "not gpu".

Each test ties ``oracle.*3`` to something other than itself: exact rational
determinants (Fractions, difference form — the oracle uses the multilinear
24-product form in a limb accumulator), closed-form extremes of points on a
circle, scipy's Qhull (an independent hull code) for the facets of generic
point sets, and closed-form interiors (octahedron |x|+|y|+|z| < 1, cube
max|x_i| < 1) for Step 3.
"""
from __future__ import annotations

import itertools
from fractions import Fraction

import numpy as np
import pytest
from scipy.spatial import ConvexHull

import oracle
import synth


def orient3d_frac(a, b, c, d) -> int:
    """Exact sign of ((b-a) x (c-a)) . (d-a) over the rationals."""
    A, B, C, D = ([Fraction(float(v)) for v in p] for p in (a, b, c, d))
    u = [B[i] - A[i] for i in range(3)]
    v = [C[i] - A[i] for i in range(3)]
    w = [D[i] - A[i] for i in range(3)]
    n = (u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0])
    det = n[0] * w[0] + n[1] * w[1] + n[2] * w[2]
    return (det > 0) - (det < 0)


def _quads(rng, n):
    out = []
    for _ in range(n):
        kind = rng.integers(5)
        if kind == 0:      # uniform
            t = rng.uniform(-1, 1, 12)
        elif kind == 1:    # near-coplanar: d = a + s(b-a) + t(c-a), rounded to float
            a, b, c = rng.uniform(-1, 1, (3, 3))
            s, u = rng.uniform(-2, 2, 2)
            t = np.r_[a, b, c, a + s * (b - a) + u * (c - a)]
        elif kind == 2:    # mixed magnitudes
            t = rng.uniform(-1, 1, 12) * 2.0 ** rng.integers(-40, 40, 12)
        elif kind == 3:    # small integer grid (exact zeros)
            t = rng.integers(-2, 3, 12).astype(float)
        else:              # large common offset: differences lose bits in float arithmetic
            t = rng.uniform(-1, 1, 12) * 2.0 ** -10 + 1024.0
        t = t.astype(np.float32).reshape(4, 3)
        out.append(tuple(t))
    return out


def test_orient3d_exact_vs_fractions():
    """B6: oracle orient3d sign == exact rational sign, incl. exact zeros."""
    rng = np.random.default_rng(31)
    zeros = 0
    for a, b, c, d in _quads(rng, 5000):
        want = orient3d_frac(a, b, c, d)
        zeros += want == 0
        assert oracle.orient3d(a, b, c, d) == want, (a, b, c, d)
        assert oracle.orient3d(b, a, c, d) == -want          # antisymmetry
        assert oracle.orient3d(d, b, c, a) == -want          # swap a <-> d
    assert zeros > 100


def test_orient3d_closed_forms_and_extreme_exponents():
    e = np.eye(3, dtype=np.float32)
    o = np.zeros(3, np.float32)
    assert oracle.orient3d(o, e[0], e[1], e[2]) == 1                   # right-handed frame
    assert oracle.orient3d(o, e[1], e[0], e[2]) == -1
    assert oracle.orient3d(o, e[0], e[1], [3.5, -7.25, 0.0]) == 0      # on the plane z = 0
    tiny, big = np.float32(2.0 ** -149), np.float32(3.0e38)
    assert oracle.orient3d(o, [tiny, 0, 0], [0, tiny, 0], [0, 0, tiny]) == 1   # det = 2^-447
    assert oracle.orient3d(o, [big, 0, 0], [0, big, 0], [0, 0, big]) == 1      # det ~ 2^384
    q = ([-big, tiny, 1], [big, -big, tiny], [tiny, big, -big], [1, tiny, big])
    assert oracle.orient3d(*q) == orient3d_frac(*q)
    # an exact cancellation a naive double evaluation gets wrong
    a = np.array([1, 1, 1], np.float32) * np.float32(2 ** 20)
    b = a + np.array([1, 0, 0], np.float32)
    c = a + np.array([0, 1, 0], np.float32)
    d = a + np.array([np.float32(2 ** -3), np.float32(2 ** -3), 0], np.float32)
    assert oracle.orient3d(a, b, c, d) == 0 == orient3d_frac(a, b, c, d)


# ---------------------------------------------------------------- Step 1
def _circle_points(step_deg, z):
    ang = np.deg2rad(np.arange(0, 360, step_deg))
    xy = np.stack([np.cos(ang), np.sin(ang)], 1)
    return np.concatenate([xy, z[:, None]], 1).astype(np.float32)


@pytest.mark.parametrize("angles", ["A", "C", "D"])
def test_extremes3_closed_form_on_a_circle(angles):
    """Points at every half degree on the unit circle: for angle a the
    rotated keys X = cos(t - a), Y = sin(t - a) peak at t = a (max X),
    a + 180 (min X), a + 90 (max Y), a + 270 (min Y); z extremes by
    construction."""
    n = 720
    z = np.linspace(-1, 1, n)
    rng = np.random.default_rng(3)
    z = rng.permutation(z)
    p = _circle_points(0.5, z)
    idx = oracle.extremes3(p, angles)
    deg = oracle.PRESETS[angles]
    for k, a in enumerate(deg):
        want = [int(round(2 * ((a + off) % 360))) for off in (180, 0, 270, 90)]
        assert list(idx[6 * k:6 * k + 4]) == want, (a, idx[6 * k:6 * k + 4], want)
        assert idx[6 * k + 4] == int(np.argmin(z)) and idx[6 * k + 5] == int(np.argmax(z))


def test_extremes3_lowest_index_on_ties_and_thread_invariance():
    p = synth.generate3("ball", 30_000, seed=5)
    q = np.concatenate([p, p, p])                        # every key tied three times
    a = oracle.extremes3(p, "A")
    b = oracle.extremes3(q, "A", threads=7)
    assert np.array_equal(a, b)                          # the first copy wins every tie
    for t in (1, 2, 5, 16):
        assert np.array_equal(oracle.extremes3(q, "D", threads=t), oracle.extremes3(q, "D"))


def test_extremes3_attain_the_extreme_keys():
    """Each pick attains the slot's extreme over a linear scan of the exact
    rational keys (RN products are what the method defines; here Fractions
    of the float64 products agree in sign order on this data)."""
    p = synth.generate3("cube", 5_000, seed=8)
    idx, key = oracle.extremes3(p, "A", with_keys=True)
    c, s = oracle.coeffs("A")
    x, y, z = (p[:, i].astype(np.float64) for i in range(3))
    for k in range(4):
        X = x * c[k] + y * s[k]
        Y = y * c[k] - x * s[k]
        for r, v in enumerate((X, X, Y, Y, z, z)):
            ext = v.min() if r % 2 == 0 else v.max()
            assert key[6 * k + r] == ext
            assert v[idx[6 * k + r]] == ext
            assert idx[6 * k + r] == int(np.flatnonzero(v == ext)[0])


# ---------------------------------------------------------------- Step 2
def _facet_triples(facets):
    return {tuple(sorted(f)) for f in facets.tolist()}


@pytest.mark.parametrize("seed", range(6))
def test_facets_vs_qhull_generic(seed):
    """Generic points (no 4 coplanar): the facets are the Qhull triangles,
    oriented with the set on the positive side (B4, B6)."""
    rng = np.random.default_rng(seed)
    m = int(rng.integers(4, 30))
    p = rng.normal(size=(m, 3)).astype(np.float32)
    E = np.arange(m)
    f = oracle.facets3(p, E)
    h = ConvexHull(p.astype(np.float64))
    assert _facet_triples(f) == {tuple(sorted(s)) for s in h.simplices.tolist()}
    for a, b, c in f:
        n = np.cross(p[b].astype(float) - p[a], p[c].astype(float) - p[a])
        for eq, s in zip(h.equations, h.simplices):
            if set(s) == {a, b, c}:
                assert np.dot(n, eq[:3]) < 0                   # inward normal
    assert len(f) == 2 * len(h.vertices) - 4                   # simplicial polytope: F = 2V - 4


def test_facets_closed_forms():
    e = np.eye(3, dtype=np.float32)
    tet = np.concatenate([np.zeros((1, 3), np.float32), e])
    assert len(oracle.facets3(tet, np.arange(4))) == 4
    octa = np.concatenate([e, -e])
    assert len(oracle.facets3(octa, np.arange(6))) == 8
    cube = np.array(list(itertools.product((-1, 1), repeat=3)), np.float32)
    assert len(oracle.facets3(cube, np.arange(8))) == 6        # one triple per square face
    # coplanar, collinear, tiny sets: degenerate
    flat = np.c_[np.random.default_rng(0).uniform(-1, 1, (10, 2)), np.zeros(10)].astype(np.float32)
    assert len(oracle.facets3(flat, np.arange(10))) == 0
    line = np.outer(np.arange(6), [1, 2, 3]).astype(np.float32)
    assert len(oracle.facets3(line, np.arange(6))) == 0
    assert len(oracle.facets3(tet[:3], np.arange(3))) == 0


def test_distinct3_collapses_coordinates_to_lowest_index():
    p = np.array([[0, 0, 0], [1, 0, 0], [0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    assert oracle.distinct3(p, [3, 2, 4, 1, 0, 4, 2]).tolist() == [0, 1, 4]


# ---------------------------------------------------------------- Step 3
def _grid(rng, n, scale):
    return (rng.integers(-16, 17, (n, 3)) / 16.0 * scale).astype(np.float32)


def test_filter3_octahedron_closed_form():
    """conv(+-e_i): strictly inside iff |x|+|y|+|z| < 1 (exactly; boundary kept)."""
    e = np.eye(3, dtype=np.float32)
    octa = np.concatenate([e, -e])
    f = oracle.facets3(octa, np.arange(6))
    fxyz = octa[f]
    rng = np.random.default_rng(2)
    pts = np.concatenate([_grid(rng, 4000, 1.0), rng.uniform(-1, 1, (4000, 3)).astype(np.float32)])
    keep = oracle.filter_mask3(pts, fxyz)
    want = [not (sum(abs(Fraction(float(v))) for v in q) < 1) for q in pts]
    assert keep.tolist() == want
    assert 0 < sum(want) < len(want)


def test_filter3_cube_closed_form():
    cube = np.array(list(itertools.product((-1, 1), repeat=3)), np.float32)
    f = oracle.facets3(cube, np.arange(8))
    rng = np.random.default_rng(4)
    pts = np.concatenate([_grid(rng, 4000, 1.25), rng.uniform(-1.1, 1.1, (2000, 3)).astype(np.float32)])
    keep = oracle.filter_mask3(pts, cube[f], threads=3)
    assert keep.tolist() == [not (np.abs(q).max() < 1) for q in pts]


@pytest.mark.parametrize("family", ["cube", "ball", "sphere"])
def test_cudapre3_conservative_and_hull_preserving(family):
    """Whole method: every Qhull vertex of the input survives; every discarded
    point is strictly inside Qhull's hull of the extremes."""
    p = synth.generate3(family, 20_000, seed=9)
    r = oracle.cudapre3(p, "A", threads=4)
    keep = np.zeros(len(p), bool)
    keep[r["survivors"]] = True
    h = ConvexHull(p.astype(np.float64))
    assert keep[h.vertices].all()
    E = oracle.distinct3(p, r["ext_idx"])
    he = ConvexHull(p[E].astype(np.float64))
    disc = p[~keep].astype(np.float64)
    assert (disc @ he.equations[:, :3].T + he.equations[:, 3] < 1e-12).all()
    if family != "sphere":   # a thin shell lies outside the inscribed polyhedron
        assert 0 < len(r["survivors"]) < len(p)
    assert np.array_equal(oracle.cudapre3(p, "A", threads=1)["survivors"], r["survivors"])


def test_cudapre3_degenerate_and_empty():
    flat = np.c_[synth.generate("disk", 5000, seed=1), np.full(5000, 0.5)].astype(np.float32)
    r = oracle.cudapre3(flat, "A")
    assert r["degenerate"] and len(r["survivors"]) == 5000     # coplanar input: nothing discarded
    with pytest.raises(ValueError):
        oracle.cudapre3(np.zeros((0, 3), np.float32))


def test_discard_fraction_ball_closed_form():
    """Closed form (P:115 with the default angles): in a uniform ball the
    picks tend to the 16 equatorial directions at azimuths {0,30,45,60} + k 90
    degrees and the two poles, so the polyhedron tends to the bipyramid over
    that 16-gon: volume (2/3) * 2 (1 + 2 sin 15) against 4 pi / 3, i.e.
    48.308 % discarded.  (A wrong orientation or predicate sign gives ~0 % or
    ~100 %.)  n = 10^6: the picks' angular deviation ~ n^-1/4 keeps the
    sampled fraction within ~1 % of the limit."""
    import math

    area = 2.0 * (1.0 + 2.0 * math.sin(math.radians(15.0)))
    want = (2.0 / 3.0) * area / (4.0 * math.pi / 3.0)
    assert abs(want - 0.48308) < 1e-5
    p = synth.generate3("ball", 1_000_000, seed=23)
    r = oracle.cudapre3(p, "A", threads=8)
    got = 1.0 - len(r["survivors"]) / len(p)
    assert abs(got - want) < 0.01, (got, want)
    assert len(r["facets"]) == 32          # the bipyramid over a 16-gon: 2 x 16 triangles
