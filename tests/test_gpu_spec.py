"""The speculative pre-filter: K1 sets aside the points
outside a region D built from the seed sample; Step 3 classifies only those
when D is verified to lie strictly inside the Step-2 polygon, else it streams
every point.  The survivors must be the oracle's either way; these tests
check both outcomes, the fallbacks and the misuse guards."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import oracle
import paper_1405_3454_b200 as cp
import synth
import synth.cuda as scuda

pytestmark = pytest.mark.gpu
THREADS = max(1, min(64, os.cpu_count() or 1))
N = 1 << 23   # >= CUDAPRE_SPEC_MIN_N


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1405_3454_b200 import build

    build.build()
    scuda.build()
    torch.cuda.set_device(0)
    yield


def _filter(xy, angles="A", ws=None):
    pts = torch.from_numpy(np.ascontiguousarray(xy)).cuda()
    ws = ws or cp.Workspace(len(xy))
    ext = cp.extremes(pts, angles, ws=ws)
    idx, sp, rep = cp.filter(pts, ext, ws=ws)
    torch.cuda.synchronize()
    return ext, idx.cpu().numpy(), sp.cpu().numpy(), cp.spec_info(ws)


def _check(xy, angles="A", want_used=None):
    ext, idx, sp, info = _filter(xy, angles)
    want = oracle.cudapre(xy, angles, threads=THREADS)
    assert ext.idx.tolist() == want["ext_idx"].tolist()
    assert np.array_equal(idx, want["survivors"])
    assert np.array_equal(sp, xy[idx])
    if want_used is not None:
        assert info["used"] == want_used, info
    return info


@pytest.mark.parametrize("family", synth.FAMILIES)
def test_spec_path_on_every_family(family):
    """Disk and Gaussian sets use the candidates (verified region); the
    near-circle set overflows its records and streams; every result exact."""
    xy = synth.generate(family, N + 12_345, seed=41)
    info = _check(xy)
    assert info["enabled"]
    if family in ("disk", "gauss"):
        assert info["used"], info
        assert info["candidates"] < 0.2 * len(xy)
    if family == "circle":
        assert not info["used"]


def test_verification_rejects_a_region_outside_the_polygon():
    """Akl-Toussaint angles (4 extremes) on a disk plus ONE far point (10, 10)
    outside the seed's sample: that point is the +x and +y extreme, so the
    Step-2 polygon is the triangle (10,10), (-1,0), (0,-1), whose edge from
    (-1,0) runs 0.67 from the centre, while the region from the sample (the
    diamond's inscribed disk, radius ~0.70) crosses it: the verification must
    fail and Step 3 stream every point."""
    xy = synth.generate("disk", N, seed=42)
    far = 2 * 1000 + 1    # pair 1000: not in a seed chunk (chunk 0 = pairs 0..127, the next ~16 k pairs on)
    xy[far] = (10.0, 10.0)
    info = _check(xy, "AT", want_used=False)
    assert info["enabled"]


def test_records_that_overflow_are_reread():
    """A run of points on the rim puts more than 56 candidates in a few
    records (re-read from the input by Step 3) while the region still holds."""
    xy = synth.generate("disk", N, seed=43)
    rim = synth.generate("circle", 40_000, seed=44, eps=0.0)
    xy[3_000_000:3_040_000] = rim
    info = _check(xy, want_used=True)
    assert info["overflow_records"] > 0


def test_candidates_are_used_once_and_only_for_their_input():
    """A second Step 3 after one Step 1 streams (the candidates were
    consumed); a Step 3 on other points than Step 1 saw streams too."""
    a = synth.generate("disk", N, seed=45)
    b = synth.generate("disk", N, seed=46)
    ws = cp.Workspace(N)
    pa, pb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    ext = cp.extremes(pa, "A", ws=ws)
    i1, _, _ = cp.filter(pa, ext, ws=ws)
    assert cp.spec_info(ws)["used"]
    i2, _, _ = cp.filter(pa, ext, ws=ws)
    assert not cp.spec_info(ws)["used"]
    assert np.array_equal(i1.cpu().numpy(), i2.cpu().numpy())
    cp.extremes(pa, "A", ws=ws)
    ib, _, _ = cp.filter(pb, ext, ws=ws)                 # points of another set, a's polygon
    assert not cp.spec_info(ws)["used"]
    ring = oracle.hull(a, oracle.extremes(a, "A"))
    want = np.flatnonzero(oracle.filter_mask(b, a[ring], threads=THREADS))
    assert np.array_equal(ib.cpu().numpy(), want)


def test_device_path_graph_and_index_base():
    """The device-resident pipeline (Step 2 on the device, verification and
    both Step-3 kernels enqueued back to back) and its CUDA graph, with a
    non-zero index_base: identical survivors, the candidates used."""
    xy = synth.generate("gauss", N + 7, seed=47)
    want = oracle.cudapre(xy, "A", threads=THREADS)["survivors"]
    pts = torch.from_numpy(xy).cuda()
    ws = cp.Workspace(len(xy))
    idx, sp, cnt = cp.pipeline(pts, "A", index_base=5, ws=ws)
    torch.cuda.synchronize()
    m = int(cnt.item())
    assert np.array_equal(idx[:m].cpu().numpy() - 5, want)
    assert cp.spec_info(ws)["used"]
    g = cp.Graph(pts, "A", ws=ws)
    for _ in range(3):
        g.launch()
    torch.cuda.synchronize()
    m = int(g.count.item())
    assert np.array_equal(g.out_idx[:m].cpu().numpy(), want)
    assert cp.spec_info(ws)["used"]
    g.close()


def test_c5_full_size_spec_matches_streaming():
    """The bench workload (2e9 disk points): the survivors with the candidates
    equal those of the streaming Step 3 element by element (the oracle check
    of the same 2e9 points is test_gpu_parity.py::test_config_c5_full)."""
    cfg = dict(synth.CONFIGS["C5"])
    n = cfg.pop("n")
    pts = scuda.generate(cfg["family"], n, seed=cfg["seed"])
    ws = cp.Workspace(n)
    cap = n // 16
    o1 = torch.empty(cap, dtype=torch.int64, device="cuda")
    o2 = torch.empty(cap, dtype=torch.int64, device="cuda")
    ext = cp.extremes(pts, "A", ws=ws)
    a, _, _ = cp.filter(pts, ext, ws=ws, out_idx=o1, return_points=False)
    assert cp.spec_info(ws)["used"]
    b, _, _ = cp.filter(pts, ext, ws=ws, out_idx=o2, return_points=False)
    assert not cp.spec_info(ws)["used"]
    assert a.shape == b.shape and bool(torch.equal(a, b))
