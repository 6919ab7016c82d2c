"""C-ABI and host-logic tests (no GPU needed).

* libcudapre.so loads and exports every function include/cudapre.h declares;
* the host-side pieces of the product (Step 2 polygon + kernel parameters,
  final hull, shard merge, angle presets) agree with the oracle / closed forms;
* the Step-3 kernel's float fast path (inner box, per-edge bounds E_j) is
  emulated EXACTLY here (fractions, correctly rounded float32 fma) on points
  hugging the polygon's edges, proving its decisions agree with the exact
  predicate before any GPU run.
"""
from __future__ import annotations

import ctypes
import os
import re
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import paper_1405_3454_b200 as cp
import synth
from tests import brute

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1405_3454_b200 import build

    build.build()
    return cp.lib()


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "cudapre.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(cudapre3?_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 11
    for name in declared:
        assert hasattr(L, name), name
    assert set(cp.SYMBOLS) == declared
    assert b"sm_100a" in L.cudapre_version()


def test_struct_sizes_match_header(L):
    # offsets derived from the C layout rules of include/cudapre.h
    assert ctypes.sizeof(cp.ExtremesT) == 8 + 8 + 32 * 8 + 32 * 8 + 32 * 8 + 8 * 8 + 8 * 8 + 8
    assert ctypes.sizeof(cp.PolygonT) == 16 + 32 * 8 + 32 * 8 + 16 + 16 + 8 + 4 * 32 * 4 + 2 * 4 * 1025
    assert ctypes.sizeof(cp.ReportT) == 64


def test_angle_presets_correctly_rounded(L):
    """Reading A5, independently of the oracle: decimal closed forms."""
    getcontext().prec = 80
    s2, s3 = Decimal(2).sqrt(), Decimal(3).sqrt()
    want = {
        "A": [(1, 0), (s3 / 2, Decimal(1) / 2), (s2 / 2, s2 / 2), (Decimal(1) / 2, s3 / 2)],
        "B": [(1, 0), (s3 / 2, Decimal(1) / 2), (s2 / 2, s2 / 2), (s2 / 2, s2 / 2)],
        "AT": [(1, 0)],
        "C": [(1, 0), ((2 + s2).sqrt() / 2, (2 - s2).sqrt() / 2), (s2 / 2, s2 / 2),
              ((2 - s2).sqrt() / 2, (2 + s2).sqrt() / 2)],
    }
    s6 = Decimal(6).sqrt()
    c15, s15 = (s6 + s2) / 4, (s6 - s2) / 4
    c225, s225 = (2 + s2).sqrt() / 2, (2 - s2).sqrt() / 2
    want["D"] = [(1, 0), (c15, s15), (c225, s225), (s3 / 2, Decimal(1) / 2), (s2 / 2, s2 / 2),
                 (Decimal(1) / 2, s3 / 2), (s225, c225), (s15, c15)]
    for name, cs in want.items():
        n, c, s = cp.angles(name)
        assert n == len(cs)
        for k, (cc, ss) in enumerate(cs):
            assert c[k] == float(Decimal(cc)) and s[k] == float(Decimal(ss)), (name, k)


def test_empty_and_bad_args_without_gpu(L):
    """Argument errors are reported before any CUDA call."""
    st = L.cudapre_extremes(None, -1, 0, 4, None, None, None, 0, None, None, None, None)
    assert st == cp.ERR_ARG
    assert b"out of range" in L.cudapre_last_error()
    bad = np.zeros(8)
    bad[0] = 0.5
    st = L.cudapre_extremes(None, 5, 0, 4, bad.ctypes.data_as(ctypes.c_void_p),
                            np.zeros(8).ctypes.data_as(ctypes.c_void_p), None, 0, None, None,
                            None, None)
    assert st == cp.ERR_ARG
    assert L.cudapre_workspace_bytes(10 ** 9) > 128 * (10 ** 9 // 16384)   # one 128-byte status line per super-tile


# ------------------------------------------------------------ host-side pieces
def _ext_from_oracle(oracle, xy, angles="A", base=0, lo=0, hi=None):
    """A cudapre_extremes_t for xy[lo:hi] built from the ORACLE's Step 1."""
    hi = len(xy) if hi is None else hi
    r = cp.ExtremesT()
    nang, c, s = cp.angles(angles)
    r.nang = nang
    r.n = hi - lo
    for k in range(32):
        r.idx[k] = -1
    for k in range(8):
        r.c[k], r.s[k] = c[k], s[k]
    if hi > lo:
        idx, key = oracle.extremes(xy[lo:hi], angles, with_keys=True)
        for k in range(4 * nang):
            r.idx[k] = int(idx[k]) + base + lo
            r.key[k] = float(key[k])
            r.pt[k].x, r.pt[k].y = map(float, xy[lo + idx[k]])
    return r


@pytest.mark.parametrize("family", ["square", "disk", "gauss", "circle"])
def test_hull_matches_oracle(L, oracle_lib, family):
    for n in (1, 2, 3, 17, 1000, 50_000):
        xy = synth.generate(family, n, seed=n)
        assert cp.hull(xy).tolist() == oracle_lib.hull(xy).tolist()
    grid = np.random.default_rng(0).integers(-3, 4, (500, 2)).astype(np.float32)
    assert cp.hull(grid).tolist() == oracle_lib.hull(grid).tolist()
    a11 = np.array([[2.0 ** -60, 0.0], [1.0, 1.0], [1 + 2.0 ** -23, 1 + 2.0 ** -23]], np.float32)
    assert cp.hull(a11).tolist() == oracle_lib.hull(a11).tolist() == [0, 2, 1]


def test_product_orient_vs_fractions(L, oracle_lib):
    """The product's exact predicate (expansions) on the oracle's hard cases,
    through the hull of 3 points (orientation sign decides the ring)."""
    rng = np.random.default_rng(11)
    from tests.test_oracle_pins import _float_triples

    for a, b, c in _float_triples(rng, 3000):
        pts = np.array([a, b, c], np.float32)
        ring = cp.hull(pts)
        assert ring.tolist() == brute.gift_wrap(pts), pts


@pytest.mark.parametrize("family", ["square", "disk", "gauss", "circle"])
@pytest.mark.parametrize("angles", ["A", "B", "C", "AT", "D"])
def test_polygon_matches_oracle(L, oracle_lib, family, angles):
    xy = synth.generate(family, 20_000, seed=5)
    ext = cp.Extremes(_ext_from_oracle(oracle_lib, xy, angles))
    poly = cp.polygon(ext)
    want = oracle_lib.polygon(xy, oracle_lib.extremes(xy, angles))
    assert poly.vidx.tolist() == want.tolist()
    assert poly.degenerate == (len(want) < 3)
    x0, x1, y0, y1 = poly.box
    if not poly.degenerate and x0 <= x1:
        ring = xy[want]
        for corner in ((x0, y0), (x1, y0), (x1, y1), (x0, y1)):
            assert brute.strictly_inside_frac(ring, corner)


def test_merge_equals_single_shard(L, oracle_lib):
    """any sharding merges to the single-set result (incl. empty shards
    and ties across shard borders)."""
    xy = np.round(synth.generate("disk", 30_001, seed=8) * 16).astype(np.float32)  # heavy ties
    whole = _ext_from_oracle(oracle_lib, xy)
    rng = np.random.default_rng(1)
    for _ in range(20):
        cuts = sorted(rng.integers(0, len(xy), rng.integers(1, 6)).tolist())
        bounds = [0, *cuts, len(xy)]
        parts = [_ext_from_oracle(oracle_lib, xy, lo=a, hi=b) for a, b in zip(bounds, bounds[1:])]
        m = cp.merge(parts)
        assert m.idx.tolist() == list(whole.idx[:16])
        assert m.n == len(xy)
    with pytest.raises(cp.CudaPreError):
        cp.merge([_ext_from_oracle(oracle_lib, xy, lo=0, hi=0)])


# ------------------------------------------------------------ K2 float path, emulated exactly
def _rn32(q: Fraction) -> np.float32:
    """Correctly rounded (nearest-even) float32 of an exact rational."""
    f = np.float32(float(q))
    best = f
    for g in (np.nextafter(f, np.float32(-np.inf)), np.nextafter(f, np.float32(np.inf))):
        if not np.isfinite(g):
            continue
        db, dg = abs(Fraction(float(best)) - q), abs(Fraction(float(g)) - q)
        if dg < db or (dg == db and (int(g.view(np.uint32)) & 1) == 0):
            best = g
    return best


def _fma32(a, b, c) -> np.float32:
    return _rn32(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def test_k2_float_decisions_are_conservative(L, oracle_lib):
    """with the library's A, B, C', E, inner box, the kernel's
    decisions (box -> discard; min g > 0 -> discard; RN(min g + 2Emax) < 0 ->
    keep) never contradict the exact predicate, on points within a few ulp of
    the polygon's edges and vertices."""
    lib = cp.lib()
    xy = synth.generate("disk", 50_000, seed=13)
    ext = _ext_from_oracle(oracle_lib, xy)
    poly = cp.PolygonT()
    assert lib.cudapre_polygon(ctypes.byref(ext), ctypes.byref(poly)) == 0
    nv = poly.nv
    V = np.array([[poly.v[j].x, poly.v[j].y] for j in range(nv)], np.float32)
    coef = [(np.float32(poly.A[j]), np.float32(poly.B[j]), np.float32(poly.C[j]), np.float32(poly.E[j]))
            for j in range(nv)]
    # E_j really bounds the float error of the kernel's expression over the bbox
    Mx = max(abs(float(xy[:, 0].min())), abs(float(xy[:, 0].max())))
    My = max(abs(float(xy[:, 1].min())), abs(float(xy[:, 1].max())))
    for j in range(nv):
        ax, ay = map(Fraction, map(float, V[j]))
        bx, by = map(Fraction, map(float, V[(j + 1) % nv]))
        A, B, C = ay - by, bx - ax, ax * by - ay * bx
        S = abs(A) * Fraction(Mx) + abs(B) * Fraction(My) + abs(C)
        assert Fraction(float(coef[j][3])) >= S * Fraction(1, 2 ** 20)
    e2max = np.float32(2 * max(c[3] for c in coef))
    assert float(e2max) == 2 * poly.err_max
    rng = np.random.default_rng(4)
    checked = decided = 0
    for j in range(nv):
        a, b = V[j].astype(np.float64), V[(j + 1) % nv].astype(np.float64)
        nrm = np.array([a[1] - b[1], b[0] - a[0]])   # inward normal (CCW ring)
        nrm /= np.hypot(*nrm)
        for t in rng.uniform(-0.05, 1.05, 40):
            base = a + t * (b - a)
            pts = []
            for d in (-3, -1, 0, 1, 3):          # within a few ulp of the edge line
                p = base.astype(np.float32)
                if d:
                    p = np.array([np.nextafter(p[0], np.float32(np.sign(d) * np.inf)), p[1]], np.float32)
                    for _ in range(abs(d) - 1):
                        p[1] = np.nextafter(p[1], np.float32(np.sign(d) * np.inf))
                pts.append(p)
            for off in (-1e-3, -1e-5, -1e-6, 1e-6, 1e-5, 1e-3):   # clearly off the line
                pts.append((base + off * nrm).astype(np.float32))
            for p in pts:
                    inside = brute.strictly_inside_frac(V, p)
                    x0, x1, y0, y1 = poly.box
                    if x0 <= p[0] <= x1 and y0 <= p[1] <= y1:
                        assert inside
                        continue
                    g = [_fma32(A, p[0], _fma32(B, p[1], Cl)) for A, B, Cl, _ in coef]
                    mn = min(g)
                    checked += 1
                    if mn > 0:
                        decided += 1
                        assert inside, p
                    elif np.float32(mn + e2max) < 0:
                        decided += 1
                        assert not inside, p
    assert checked > 1000 and decided > 0.3 * checked   # ~5/11 of the probes sit in the band


def test_k2_inner_disk_is_conservative(L, oracle_lib):
    """every point the kernel's disk test accepts
    (RN32(RN32(dx*dx) + RN32(dy*dy)) < r2, dx = RN32(x - ox)) is strictly inside
    the ring by the exact predicate — probed on and around the disk boundary."""
    for family, seed in (("disk", 13), ("square", 2), ("gauss", 4), ("circle", 5)):
        xy = synth.generate(family, 50_000, seed=seed)
        ext = _ext_from_oracle(oracle_lib, xy)
        poly = cp.polygon(cp.Extremes(ext))
        ox, oy, r2 = poly.circle
        if r2 < 0:
            assert family == "circle" or poly.degenerate
            continue
        V = poly.v
        r = float(np.sqrt(np.float64(r2)))
        rng = np.random.default_rng(seed)
        accepted = 0
        for th in rng.uniform(0, 2 * np.pi, 400):
            for f in (0.999, 0.99999, 1.0, 1.000001, 1.00001):
                p = np.array([ox + f * r * np.cos(th), oy + f * r * np.sin(th)], np.float32)
                dx = np.float32(p[0] - np.float32(ox))
                dy = np.float32(p[1] - np.float32(oy))
                d2 = np.float32(np.float32(dx * dx) + np.float32(dy * dy))   # kernel: FADD2, FMUL2, FADD
                if d2 < np.float32(r2):
                    accepted += 1
                    assert brute.strictly_inside_frac(V, p), (family, p)
        assert accepted > 400


def _prescreen_params(T, c, s):
    """Python mirror of k1_extremes.cu:prescreen_params (float32/float64 IEEE ops)."""
    f32 = np.float32
    cx = f32(f32(f32(T[0]) + f32(T[1])) * f32(0.5))
    cy = f32(f32(f32(T[2]) + f32(T[3])) * f32(0.5))
    smin = np.inf
    for k in range(len(c)):
        px = float(cx) * c[k] + float(cy) * s[k]
        py = float(cy) * c[k] - float(cx) * s[k]
        smin = min(smin, px - float(T[4 * k]), float(T[4 * k + 1]) - px,
                   py - float(T[4 * k + 2]), float(T[4 * k + 3]) - py)
    ac = abs(float(cx)) + abs(float(cy))
    rho = smin * (1.0 - 2.0 ** -10) - ac * 2.0 ** -17 - 2.0 ** -100
    if not rho > 0:
        return cx, cy, np.float32(-1.0)
    r2 = min(rho * rho * (1.0 - 2.0 ** -16), 2.0 ** 126)
    f = np.float32(r2)
    if float(f) > r2:
        f = np.nextafter(f, np.float32(0))
    return cx, cy, f


@pytest.mark.parametrize("family", ["disk", "square", "gauss", "circle"])
def test_k1_prescreen_is_conservative(L, oracle_lib, family):
    """with thresholds T that are safe float roundings of real
    extreme keys, every point the pre-screen rejects (float d2 < rho2) has
    exact binary64 keys strictly worse than every threshold, so it can never be
    an extreme.  Probed on points straddling the pre-screen circle."""
    xy = synth.generate(family, 40_000, seed=17)
    c, s = oracle_lib.coeffs("A")
    _, keys = oracle_lib.extremes(xy, "A", with_keys=True)
    # thresholds as the kernel holds them: max slots RD32, min slots RU32 of real keys
    T = []
    for k, v in enumerate(keys):
        f = np.float32(v)
        if k % 2 == 1 and float(f) > v:
            f = np.nextafter(f, np.float32(-np.inf))
        if k % 2 == 0 and float(f) < v:
            f = np.nextafter(f, np.float32(np.inf))
        T.append(f)
    cx, cy, rho2 = _prescreen_params(T, c, s)
    assert rho2 > 0
    r = float(np.sqrt(np.float64(rho2)))
    rng = np.random.default_rng(3)
    th = rng.uniform(0, 2 * np.pi, 20_000)
    f = rng.uniform(0.999, 1.001, 20_000)
    pts = np.stack([float(cx) + f * r * np.cos(th), float(cy) + f * r * np.sin(th)], 1).astype(np.float32)
    d = (pts - np.array([cx, cy], np.float32)).astype(np.float32)
    d2 = (d[:, 0] * d[:, 0]).astype(np.float32) + (d[:, 1] * d[:, 1]).astype(np.float32)
    rejected = pts[d2.astype(np.float32) < rho2]
    assert len(rejected) > 1000
    P = rejected.astype(np.float64)
    for k in range(4):
        X = P[:, 0] * c[k] + P[:, 1] * s[k]
        Y = P[:, 1] * c[k] - P[:, 0] * s[k]
        assert (X > float(T[4 * k])).all() and (X < float(T[4 * k + 1])).all()
        assert (Y > float(T[4 * k + 2])).all() and (Y < float(T[4 * k + 3])).all()


@pytest.mark.parametrize("family", ["disk", "square", "gauss", "circle"])
def test_k2_sector_table_is_conservative(L, oracle_lib, family):
    """every probe the kernel's sector test accepts
    (RN32(RN32(dx^2)+RN32(dy^2)) < sector_r2[round(256 pa)], pa = pseudo-angle
    of RN32(p - c)) is strictly inside the ring by the exact predicate; probes
    sit at radius sqrt(sector_r2) * (1 +- a few ulp) in every bucket."""
    import time

    xy = synth.generate(family, 50_000, seed=29)
    ext = _ext_from_oracle(oracle_lib, xy)
    t0 = time.perf_counter()
    poly = cp.polygon(cp.Extremes(ext))
    dt = time.perf_counter() - t0
    assert dt < 0.05, dt                                  # host Step 2 stays cheap
    sr2 = np.frombuffer(poly.raw.sector_r2, np.float32)
    ox, oy = np.float32(poly.circle[0]), np.float32(poly.circle[1])
    assert (sr2 > 0).all()
    V = poly.v
    rng = np.random.default_rng(7)
    pa = rng.uniform(0, 4, 6000)
    t = np.where(pa <= 2, pa - 1, 3 - pa)
    ux = np.where(pa <= 2, 1 - np.abs(t), -(1 - np.abs(t)))
    u = np.stack([ux, t], 1) / np.hypot(ux, t)[:, None]
    b0 = np.clip(np.round(256 * pa).astype(int), 0, 1024)
    f = rng.choice([1 - 1e-6, 1 - 1e-7, 1.0, 1 + 1e-7], len(pa))
    r = np.sqrt(sr2[b0].astype(np.float64)) * f
    pts = (np.array([ox, oy], np.float64) + r[:, None] * u).astype(np.float32)
    d = (pts - np.array([ox, oy], np.float32)).astype(np.float32)
    d2 = (d[:, 0] * d[:, 0]).astype(np.float32) + (d[:, 1] * d[:, 1]).astype(np.float32)
    tt = d[:, 1].astype(np.float64) / (np.abs(d[:, 0]).astype(np.float64) + np.abs(d[:, 1]))
    pe = np.where(d[:, 0] >= 0, tt + 1, 3 - tt)
    b = np.clip(np.round(256 * pe).astype(int), 0, 1024)
    acc = d2.astype(np.float32) < sr2[b]
    assert acc.sum() > 1000
    for p in pts[acc][:1500]:
        assert brute.strictly_inside_frac(V, p), (family, p)
    # outer table: probes just beyond sqrt(sector_out_r2) classified "outside"
    # must not be strictly inside (the kernel keeps them without edge tests)
    so2 = np.frombuffer(poly.raw.sector_out_r2, np.float32)
    assert np.isfinite(so2).all() and (so2 >= sr2).all()
    r = np.sqrt(so2[b0].astype(np.float64)) * rng.choice([1 + 1e-6, 1 + 1e-7, 1.0, 1 - 1e-7], len(pa))
    pts = (np.array([ox, oy], np.float64) + r[:, None] * u).astype(np.float32)
    d = (pts - np.array([ox, oy], np.float32)).astype(np.float32)
    d2 = (d[:, 0] * d[:, 0]).astype(np.float32) + (d[:, 1] * d[:, 1]).astype(np.float32)
    tt = d[:, 1].astype(np.float64) / (np.abs(d[:, 0]).astype(np.float64) + np.abs(d[:, 1]))
    pe = np.where(d[:, 0] >= 0, tt + 1, 3 - tt)
    b = np.clip(np.round(256 * pe).astype(int), 0, 1024)
    out = d2.astype(np.float32) > so2[b]
    assert out.sum() > 1000
    for p in pts[out][:1500]:
        assert not brute.strictly_inside_frac(V, p), (family, p)


@pytest.mark.parametrize("family", ["disk", "square", "gauss", "circle"])
@pytest.mark.parametrize("angles", ["A", "D"])
def test_k2_candidate_edges_hold_the_exit_edge(L, oracle_lib, family, angles):
    """for every bucket a probe's ray can land in (its exact
    pseudo-angle bucket +- the kernel's error, < 2^-12 bucket), the bucket's
    candidate-edge range (sedge) holds the edge the ray from the centre exits
    through — decided exactly with rationals on the probe's float coordinates
    (a ray through a vertex may use either adjacent edge)."""
    from fractions import Fraction as Fr

    xy = synth.generate(family, 50_000, seed=31)
    ext = cp.Extremes(_ext_from_oracle(oracle_lib, xy, angles))
    g = cp.geometry(ext)
    nv = int(np.frombuffer(g[:4], np.int32)[0])
    ox, oy = np.frombuffer(g[32:40], np.float32)
    vx = np.frombuffer(g[432:432 + 132], np.float32)[:nv]
    vy = np.frombuffer(g[564:564 + 132], np.float32)[:nv]
    sedge = np.frombuffer(g[8896:8896 + 2 * 1025], np.uint16)
    assert nv >= 3 and (sedge != 0xFFFF).mean() > 0.9
    c = (Fr(float(ox)), Fr(float(oy)))
    V = [(Fr(float(a)), Fr(float(b))) for a, b in zip(vx, vy)]

    def cross(ax, ay, bx, by):
        return ax * by - ay * bx

    rng = np.random.default_rng(3)
    pa = rng.uniform(0, 4, 1500)
    t = np.where(pa <= 2, pa - 1, 3 - pa)
    u = np.stack([np.where(pa <= 2, 1 - np.abs(t), -(1 - np.abs(t))), t], 1)
    pts = (np.array([ox, oy], np.float64) + rng.uniform(0.5, 1.5, (len(pa), 1)) * u).astype(np.float32)
    checked = 0
    for p in pts:
        dx, dy = Fr(float(p[0])) - c[0], Fr(float(p[1])) - c[1]
        if dx == 0 and dy == 0:
            continue
        # exit edges: j with the direction in the closed wedge (v_j - c, v_j+1 - c)
        exits = set()
        for j in range(nv):
            k = (j + 1) % nv
            s0 = cross(V[j][0] - c[0], V[j][1] - c[1], dx, dy)
            s1 = cross(V[k][0] - c[0], V[k][1] - c[1], dx, dy)
            if s0 >= 0 and s1 <= 0:
                exits.add(j)
        assert exits
        pe = float(dy / (abs(dx) + abs(dy)))
        pe = pe + 1 if dx >= 0 else 3 - pe
        for b in range(int(np.floor(256 * pe - 0.5 - 2 ** -10)), int(np.ceil(256 * pe + 0.5 + 2 ** -10)) + 1):
            if abs(b - 256 * pe) > 0.5 + 2 ** -10:
                continue
            for bb in {b % 1024, b % 1024 + (1024 if b % 1024 == 0 else 0)}:
                if bb > 1024 or sedge[bb] == 0xFFFF:
                    continue
                lo, hi = int(sedge[bb]) & 0xFF, int(sedge[bb]) >> 8
                rng_edges = {(lo + i) % nv for i in range((hi - lo) % nv + 1)}
                assert exits & rng_edges, (family, angles, bb, lo, hi, exits)
                checked += 1
    assert checked > 1000


def test_filtered_orient_in_step2_vs_fractions(L, oracle_lib):
    """The Step-2 builders use a float32 orientation filter in front of the
    exact predicate (exact.cuh orient_sign_filtered); on the oracle's hard
    triples (near-collinear, subnormal, huge) the polygon's ring must equal
    the exact gift wrap."""
    rng = np.random.default_rng(12)
    from tests.test_oracle_pins import _float_triples

    checked = 0
    for a, b, c in _float_triples(rng, 3000):
        pts = np.array([a, b, c], np.float32)
        if not np.isfinite(pts).all():
            continue
        r = cp.ExtremesT()
        r.nang, r.n = 1, 3
        for k in range(32):
            r.idx[k] = -1
        r.c[0], r.s[0] = 1.0, 0.0
        for slot, i in enumerate((0, 1, 2, 0)):
            r.idx[slot] = i
            r.pt[slot].x, r.pt[slot].y = float(pts[i, 0]), float(pts[i, 1])
        poly = cp.polygon(cp.Extremes(r))
        want = brute.gift_wrap(pts)
        if len(want) >= 3:
            assert poly.vidx.tolist() == want, pts
            checked += 1
        else:
            assert poly.degenerate, pts
    assert checked > 500


def test_plain_c_client_compiles_links_and_runs(tmp_path):
    """The boundary is a C ABI: include/cudapre.h compiles as strict C99 and a
    C program links against libcudapre.so and calls host-only entry points
    (2D and 3D) — no torch, no C++ in the caller."""
    import subprocess

    src = tmp_path / "client.c"
    src.write_text(r"""
#include <stdio.h>
#include "cudapre.h"
int main(void) {
    int32_t nang = 0; double c[8], s[8];
    if (cudapre_angles_preset(0, &nang, c, s) != CUDAPRE_OK || nang != 4) return 1;
    if (cudapre_workspace_bytes(1000) == 0 || cudapre3_workspace_bytes(1000) == 0) return 2;
    float a[3] = {0, 0, 0}, b[3] = {1, 0, 0}, cc[3] = {0, 1, 0}, d[3] = {0, 0, 1};
    if (cudapre3_orient(a, b, cc, d) != 1 || cudapre3_orient(a, cc, b, d) != -1) return 3;
    cudapre_pt pts[4] = {{0, 0}, {1, 0}, {0, 1}, {0.25f, 0.25f}};
    int64_t ring[4], len = 0;
    if (cudapre_hull(pts, NULL, 4, ring, &len) != CUDAPRE_OK || len != 3) return 4;
    printf("ok %s\n", cudapre_version());
    return 0;
}
""")
    exe = tmp_path / "client"
    libdir = os.path.dirname(cp.LIB_PATH)
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-pedantic", f"-I{ROOT}/include", str(src),
                           f"-L{libdir}", "-lcudapre", f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.startswith("ok "), (out.returncode, out.stdout, out.stderr)
