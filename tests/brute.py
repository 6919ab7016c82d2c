"""Brute-force exact references used to PIN the oracle (test tree only).

Everything here uses Python ``fractions.Fraction`` on the exact values of the
float32 inputs, so it shares no arithmetic with either the oracle (C limb
accumulator) or the CUDA path (floating-point expansions).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def F(v) -> Fraction:
    return Fraction(float(np.float32(v)))


def orient_frac(a, b, c) -> int:
    ax, ay, bx, by, cx, cy = map(F, (*a, *b, *c))
    d = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)
    return (d > 0) - (d < 0)


def gift_wrap(pts, ids=None) -> list[int]:
    """Jarvis march with exact orientation (SPEC.md:226's independent oracle).

    Canonical ring: CCW from the lexicographically smallest point, collinear
    points excluded, duplicate coordinates represented by their lowest id."""
    pts = np.asarray(pts, np.float32).reshape(-1, 2)
    if ids is None:
        ids = list(range(len(pts)))
    # dedup coordinates keeping lowest id
    best = {}
    for i in ids:
        key = (float(pts[i, 0]) + 0.0, float(pts[i, 1]) + 0.0)  # -0 == +0
        if key not in best or i < best[key]:
            best[key] = i
    cand = sorted(best.values(), key=lambda i: (float(pts[i, 0]), float(pts[i, 1])))
    if len(cand) <= 1:
        return cand
    P = {i: (F(pts[i, 0]), F(pts[i, 1])) for i in cand}

    def orient(a, b, c):
        (ax, ay), (bx, by), (cx, cy) = P[a], P[b], P[c]
        d = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)
        return (d > 0) - (d < 0)

    def dist2(a, b):
        (ax, ay), (bx, by) = P[a], P[b]
        return (ax - bx) ** 2 + (ay - by) ** 2

    start = cand[0]
    ring = [start]
    cur = start
    while True:
        nxt = None
        for q in cand:
            if q == cur:
                continue
            if nxt is None:
                nxt = q
                continue
            o = orient(cur, nxt, q)
            # q is more clockwise than nxt -> take q; collinear -> farther
            if o < 0 or (o == 0 and dist2(cur, q) > dist2(cur, nxt)):
                nxt = q
        if nxt == start or nxt is None:
            break
        ring.append(nxt)
        cur = nxt
        if len(ring) > len(cand):
            raise RuntimeError("gift wrapping did not close")
    if len(ring) == 2:
        return ring
    # all-collinear input: the march goes out and comes back; keep endpoints
    if all(orient(ring[0], ring[1], r) == 0 for r in ring[2:]):
        return [ring[0], max(ring, key=lambda r: dist2(ring[0], r))]
    return ring


def strictly_inside_frac(ring_xy, p) -> bool:
    ring_xy = np.asarray(ring_xy, np.float32).reshape(-1, 2)
    nv = len(ring_xy)
    if nv < 3:
        return False
    return all(orient_frac(ring_xy[j], ring_xy[(j + 1) % nv], p) > 0 for j in range(nv))


def is_hull_vertex_bruteforce(pts, i) -> bool:
    """O(n^3): p_i is a strictly convex hull vertex iff it is not in any
    closed triangle / segment of the other (distinct) points."""
    pts = np.asarray(pts, np.float32).reshape(-1, 2)
    p = tuple(map(float, pts[i]))
    others = {(float(x) + 0.0, float(y) + 0.0) for j, (x, y) in enumerate(pts)}
    others.discard((p[0] + 0.0, p[1] + 0.0))
    others = list(others)
    n = len(others)

    def on_segment(a, b, q):
        if orient_frac(a, b, q) != 0:
            return False
        return (min(a[0], b[0]) <= q[0] <= max(a[0], b[0])
                and min(a[1], b[1]) <= q[1] <= max(a[1], b[1]))

    for a in range(n):
        for b in range(a + 1, n):
            if on_segment(others[a], others[b], p):
                return False
            for c in range(b + 1, n):
                o1 = orient_frac(others[a], others[b], p)
                o2 = orient_frac(others[b], others[c], p)
                o3 = orient_frac(others[c], others[a], p)
                if orient_frac(others[a], others[b], others[c]) == 0:
                    continue
                if (o1 >= 0 and o2 >= 0 and o3 >= 0) or (o1 <= 0 and o2 <= 0 and o3 <= 0):
                    return False
    return True


def extremes_numpy(pts, c, s) -> np.ndarray:
    """Step 1 by numpy float64 elementwise ops (IEEE, no contraction) and
    first-occurrence argmin/argmax — an independent library implementation."""
    p = np.asarray(pts, np.float32).reshape(-1, 2).astype(np.float64)
    x, y = p[:, 0], p[:, 1]
    out = []
    for ck, sk in zip(c, s):
        X = x * ck + y * sk
        Y = y * ck - x * sk
        out += [np.argmin(X), np.argmax(X), np.argmin(Y), np.argmax(Y)]
    return np.asarray(out, np.int64)
