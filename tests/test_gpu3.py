"""GPU parity of the 3D extension: K1-3D picks, the
host polyhedron and K2-3D survivors must equal the oracle's exactly, at
sizes that span many tiles with ragged tails, for aligned and misaligned
inputs, ties, degenerate and extreme-magnitude inputs; at large sizes the
picks are compared exactly and the classification on a sample."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1405_3454_b200 as cp
import synth
import synth.cuda

pytestmark = pytest.mark.gpu

THREADS = max(1, min(64, os.cpu_count() or 1))


def _run(xyz, angles="A", index_base=0, view_offset=0, flags=0):
    if view_offset:
        full = torch.from_numpy(np.ascontiguousarray(np.concatenate([np.zeros((view_offset, 3), np.float32),
                                                                       xyz]))).cuda()
        pts = full[view_offset:]
    else:
        pts = torch.from_numpy(np.ascontiguousarray(xyz)).cuda()
    ext = cp.extremes3(pts, angles, index_base=index_base)
    idx, sp, poly = cp.filter3(pts, ext, index_base=index_base, flags=flags)
    torch.cuda.synchronize()
    assert poly.raw.empty_cells == 0   # the direction-cell fail-safe never fires
    return ext, idx.cpu().numpy(), sp.cpu().numpy(), poly


def _check(xyz, angles="A", **kw):
    ext, idx, sp, poly = _run(xyz, angles, **kw)
    base = kw.get("index_base", 0)
    want = oracle.cudapre3(xyz, angles, threads=THREADS)
    assert (ext.idx - base).tolist() == want["ext_idx"].tolist()
    assert (poly.facets - base).tolist() == want["facets"].tolist()
    assert np.array_equal(idx - base, want["survivors"])
    assert np.array_equal(sp, xyz[want["survivors"]])
    return ext, idx, poly


@pytest.mark.parametrize("family", ["cube", "ball", "sphere"])
@pytest.mark.parametrize("angles", ["A", "AT", "C", "D"])
@pytest.mark.parametrize("n", [5, 1_001, 300_007])
def test_parity_families_angles_sizes(family, angles, n):
    _check(synth.generate3(family, n, seed=n % 53 + 1), angles)


@pytest.mark.parametrize("n", [2_000_003, 4_194_305])
def test_parity_many_tiles(n):
    _check(synth.generate3("ball", n, seed=7))


def test_misaligned_and_index_base():
    xyz = synth.generate3("cube", 500_001, seed=2)
    _check(xyz, view_offset=1)                 # 12-byte offset: scalar loads
    _check(xyz, index_base=123_456_789_012)


def test_ties_lattice_duplicates_offsets():
    rng = np.random.default_rng(8)
    cases = [
        rng.integers(-3, 4, (200_001, 3)).astype(np.float32),                       # coplanar faces, ties
        np.round(synth.generate3("ball", 300_001, seed=1) * 16).astype(np.float32),  # heavy ties
        (synth.generate3("ball", 200_001, seed=3) + np.float32(1e4)).astype(np.float32),   # large offset
        (synth.generate3("cube", 100_001, seed=4).astype(np.float64) * 1e-30).astype(np.float32),
        (synth.generate3("cube", 100_001, seed=5).astype(np.float64) * 1e30).astype(np.float32),
        np.tile(np.float32([[0.5, -0.25, 2.0]]), (70_001, 1)),                       # one distinct point
    ]
    for xyz in cases:
        _check(xyz)


def test_degenerate_coplanar_keeps_everything():
    xy = synth.generate("disk", 100_003, seed=6)
    xyz = np.c_[xy, np.float32(0.5) * xy[:, 0]].astype(np.float32)   # exactly on the plane z = x / 2
    ext, idx, poly = _check(xyz)
    assert poly.degenerate and len(idx) == len(xyz)


def test_errors():
    with pytest.raises(cp.CudaPreError) as e:
        cp.extremes3(torch.empty((0, 3), device="cuda"))
    assert e.value.status == cp.ERR_EMPTY
    xyz = synth.generate3("ball", 10_000, seed=1)
    xyz[777, 2] = np.nan
    with pytest.raises(cp.CudaPreError) as e:
        cp.extremes3(torch.from_numpy(xyz).cuda())
    assert e.value.status == cp.ERR_NONFINITE


def test_workspace_reuse_across_sizes():
    ws = cp.Workspace3(3_000_000)
    for n, seed in ((3_000_000, 1), (10_001, 2), (2_500_000, 3), (1, 4), (3_000_000, 5)):
        xyz = synth.generate3("ball", n, seed=seed)
        pts = torch.from_numpy(xyz).cuda()
        ext = cp.extremes3(pts, "A", ws=ws)
        idx, _, _ = cp.filter3(pts, ext, ws=ws, return_points=False)
        want = oracle.cudapre3(xyz, "A", threads=THREADS)
        assert np.array_equal(idx.cpu().numpy(), want["survivors"])


def test_cuda_generator_matches_numpy():
    for fam in synth.FAMILIES3:
        a = synth.cuda.generate3(fam, 300_001, seed=11, base=5).cpu().numpy()
        b = synth.generate3(fam, 300_001, seed=11, base=5)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), fam


def test_large_sampled():
    """Bench-scale input generated on the device: picks equal the oracle's
    exactly; survivors ascend; the classification of 50k sampled points
    equals the oracle's against the oracle's own polyhedron."""
    n = 200_000_000
    pts = synth.cuda.generate3("ball", n, seed=23)
    ext = cp.extremes3(pts, "A")
    idx, _, poly = cp.filter3(pts, ext, return_points=False)
    torch.cuda.synchronize()
    host = pts.cpu().numpy()
    want_ext = oracle.extremes3(host, "A", threads=THREADS)
    assert ext.idx.tolist() == want_ext.tolist()
    E = oracle.distinct3(host, want_ext)
    F = oracle.facets3(host, E)
    assert poly.facets.tolist() == F.tolist()
    got = idx.cpu().numpy()
    assert np.all(np.diff(got) > 0)
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(n, 50_000, replace=False))
    keep = oracle.filter_mask3(host[sample], host[F], threads=THREADS)
    assert np.array_equal(np.isin(sample, got), keep)
    del host


def test_every_facet_path():
    """Without direction cells (the host's fallback when the rounded centre is
    not strictly inside) every point goes through the warp-cooperative pass
    over all facets: the same survivors."""
    for fam, n in (("ball", 300_007), ("cube", 100_003)):
        ext, idx, poly = _check(synth.generate3(fam, n, seed=31), flags=cp.FLAG3_NO_CELLS)
        assert poly.raw.cells == 0


def test_capacity_error_writes_the_first_survivors():
    """CAPACITY when the survivors exceed the buffer: the first `capacity`
    survivors (ascending) are still written, and the error says so."""
    xyz = synth.generate3("cube", 200_003, seed=12)
    pts = torch.from_numpy(xyz).cuda()
    ext = cp.extremes3(pts, "A")
    want = oracle.cudapre3(xyz, "A", threads=THREADS)["survivors"]
    cap = len(want) // 3
    out_idx = torch.full((cap,), -7, dtype=torch.int64, device="cuda")
    with pytest.raises(cp.CudaPreError) as e:
        cp.filter3(pts, ext, out_idx=out_idx, return_points=False)
    assert e.value.status == cp.ERR_CAPACITY
    torch.cuda.synchronize()
    assert np.array_equal(out_idx.cpu().numpy(), want[:cap])


@pytest.mark.parametrize("sub,deg", [((0, 2), (0.0, 45.0)), ((0, 1, 3), (0.0, 30.0, 60.0)), ((0, 1, 2, 2), (0.0, 30.0, 45.0, 45.0))])
def test_parity_two_three_and_repeated_angles(sub, deg):
    """The 2- and 3-angle kernels and a repeated angle (the paper's literal
    {0, 30, 45, 45}): the product takes slices of its own preset
    coefficients, the oracle its own table for the same degrees."""
    _, c, s = cp.angles("A")
    ang = (c[list(sub)], s[list(sub)])
    xyz = synth.generate3("ball", 250_003, seed=len(sub) + 40)
    pts = torch.from_numpy(xyz).cuda()
    ext = cp.extremes3(pts, ang)
    idx, _, poly = cp.filter3(pts, ext, return_points=False)
    want = oracle.cudapre3(xyz, deg, threads=THREADS)
    assert ext.idx.tolist() == want["ext_idx"].tolist()
    assert poly.facets.tolist() == want["facets"].tolist()
    assert np.array_equal(idx.cpu().numpy(), want["survivors"])


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 2047, 2048, 2049, 4095, 4096, 4097, 6143, 6145, 8191, 131_073])
def test_parity_tile_and_quad_boundaries(n):
    """Sizes at the 4-point quad and 2048-point tile boundaries (ragged tails,
    a last tile with one point, exactly full tiles), aligned and misaligned."""
    xyz = synth.generate3("cube", n, seed=n % 29 + 3)
    _check(xyz)
    if n >= 4:
        _check(xyz, view_offset=1, index_base=5)


def test_k1_screen_near_ties_and_exact_ties():
    """K1-3D's float screen (quad-level margin): 10^6 points
    on a unit circle in the xy-plane — near every rotated extreme many keys
    lie within the float margin of each other, so the exact binary64 path
    decides — plus exact copies of points at higher indices (ties: lowest
    index wins) and a scaled, offset copy of the whole set."""
    n = 1_000_000
    t = np.arange(n, dtype=np.float64) * (2 * np.pi / n)
    rng = np.random.default_rng(21)
    base = np.stack([np.cos(t), np.sin(t), rng.uniform(-1, 1, n)], 1).astype(np.float32)
    dup = base[rng.integers(0, n, 200_000)]
    for xyz in (np.concatenate([base, dup]),
                (np.concatenate([base, dup]).astype(np.float64) * 3e5 + 7e5).astype(np.float32)):
        pts = torch.from_numpy(np.ascontiguousarray(xyz)).cuda()
        for angles in ("A", "D"):
            got = cp.extremes3(pts, angles).idx
            want = oracle.extremes3(xyz, angles, threads=THREADS)
            assert got.tolist() == want.tolist(), angles


@pytest.mark.parametrize("k", [2, 3, 8])
def test_sharded_pipeline(k):
    """k contiguous shards (what k ranks hold): per-shard K1-3D with global
    indices, the merged Step-1 blocks, per-shard K2-3D: the concatenated
    survivors are the oracle's single-set answer (ties across cuts: heavy
    rounding)."""
    xyz = np.round(synth.generate3("ball", 600_007, seed=19) * 64).astype(np.float32)
    n = len(xyz)
    cuts = [n * r // k for r in range(k + 1)]
    parts, shards = [], []
    for r in range(k):
        lo, hi = cuts[r], cuts[r + 1]
        pts = torch.from_numpy(np.ascontiguousarray(xyz[lo:hi])).cuda()
        ws = cp.Workspace3(hi - lo)
        parts.append(cp.extremes3(pts, "A", index_base=lo, ws=ws))
        shards.append((pts, ws, lo))
    merged = cp.merge3(parts)
    want = oracle.cudapre3(xyz, "A", threads=THREADS)
    assert merged.idx.tolist() == want["ext_idx"].tolist()
    got = []
    for pts, ws, lo in shards:
        idx, sp, poly = cp.filter3(pts, merged, index_base=lo, ws=ws)
        assert poly.facets.tolist() == want["facets"].tolist()
        got.append(idx.cpu().numpy())
    assert np.array_equal(np.concatenate(got), want["survivors"])


def test_degenerate_collinear_keeps_everything():
    """All points on one line (exactly representable direction): every
    triple is collinear, there is no facet, nothing is inside."""
    t = np.random.default_rng(4).integers(-1000, 1001, 50_003).astype(np.float32) / np.float32(8)
    xyz = np.stack([t, np.float32(2) * t, np.float32(-0.5) * t], 1).astype(np.float32)
    ext, idx, poly = _check(xyz)
    assert poly.degenerate and len(idx) == len(xyz)
