"""Final hull on the GPU: the ring from cudapre_hull_device
must equal the host monotone chain on the survivors and the oracle's hull of
the whole input (the hull of the survivors is the hull of
the set because Step 3 only drops points strictly inside a polygon of input
points)."""
import ctypes
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1405_3454_b200 as cp
import synth

pytestmark = pytest.mark.gpu

THREADS = max(1, min(64, os.cpu_count() or 1))


def _check(xy, angles="A", oracle_hull=True):
    pts = torch.from_numpy(np.ascontiguousarray(xy)).cuda()
    idx, sp, rep = cp.cuda_pre(pts, angles)
    m = idx.shape[0]
    ring, remaining = cp.hull_device(sp, idx, m, rep["polygon"], return_remaining=True)
    host = cp.hull(xy, idx.cpu().numpy())
    assert ring.tolist() == host.tolist()
    if oracle_hull:
        assert ring.tolist() == oracle.hull(xy).tolist()
    return m, remaining, ring


@pytest.mark.parametrize("family", ["square", "disk", "gauss", "circle"])
@pytest.mark.parametrize("n", [1_001, 200_003, 2_000_003])
def test_hull_device_matches_host_and_oracle(family, n):
    xy = synth.generate(family, n, seed=n % 89 + 3)
    m, remaining, ring = _check(xy, oracle_hull=n <= 200_003)
    assert len(ring) >= 3
    assert remaining <= m


def test_hull_device_prunes_large_inputs():
    """The second filter leaves a small fraction of the survivors."""
    xy = synth.generate("disk", 4_000_037, seed=5)
    m, remaining, _ = _check(xy, oracle_hull=False)
    assert remaining < 0.02 * m, (remaining, m)


def test_hull_device_ties_lattice_offsets_and_degenerate():
    rng = np.random.default_rng(9)
    cases = [
        np.round(synth.generate("disk", 300_001, seed=1) * 32).astype(np.float32),   # duplicates on the hull
        rng.integers(-50, 51, (200_001, 2)).astype(np.float32),                      # lattice: collinear hull points
        (synth.generate("gauss", 300_001, seed=2) + np.float32(1e4)).astype(np.float32),
        np.stack([np.linspace(-1, 1, 5_001), np.linspace(-1, 1, 5_001)], 1).astype(np.float32),   # degenerate
    ]
    for xy in cases:
        _check(xy)


def test_hull_device_after_device_pipeline():
    """Survivors and polygon from the device-resident path (f3)."""
    xy = synth.generate("disk", 1_000_003, seed=12)
    pts = torch.from_numpy(xy).cuda()
    ws = cp.Workspace(len(xy))
    out_idx, out_pts, count = cp.pipeline(pts, "A", ws=ws)
    torch.cuda.synchronize()
    m = int(count.item())
    raw = cp.PolygonT.from_buffer_copy(
        ws.tensor[cp.WS_POLY_OFFSET:cp.WS_POLY_OFFSET + ctypes.sizeof(cp.PolygonT)].cpu().numpy().tobytes())
    ring = cp.hull_device(out_pts, out_idx, m, raw)
    assert ring.tolist() == oracle.hull(xy).tolist()


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 33, 4_097])
@pytest.mark.parametrize("angles", ["A", "D"])
def test_hull_device_tiny_inputs(n, angles):
    """Tiny sets (a single point, two, collinear triples, sets where every
    point is an extreme) through Steps 1-3 and the GPU hull, for the default
    and the 8-angle preset (up to 32-vertex polygons)."""
    for family in ("square", "disk", "circle"):
        xy = synth.generate(family, n, seed=100 + n)
        _check(xy, angles)
    dup = np.repeat(synth.generate("disk", max(1, n // 3), seed=7), 3, axis=0)[:n]   # exact duplicates
    _check(np.ascontiguousarray(dup), angles)
