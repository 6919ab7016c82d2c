"""Device-resident Steps 2-3: the polygon and the Step-3
geometry built on the device must equal the host build byte for byte, and
the device path (filter_device, pipeline, CUDA graph) must return exactly the
oracle's survivors — the same bar as the host path (tests/test_gpu_parity.py).
"""
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


def _device_pages(ws, nbytes_geom):
    t = ws.tensor
    geom = bytes(t[cp.WS_GEOM_OFFSET:cp.WS_GEOM_OFFSET + nbytes_geom].cpu().numpy().tobytes())
    psz = ctypes.sizeof(cp.PolygonT)
    poly = bytes(t[cp.WS_POLY_OFFSET:cp.WS_POLY_OFFSET + psz].cpu().numpy().tobytes())
    return geom, poly


@pytest.mark.parametrize("family", ["square", "disk", "gauss", "circle"])
@pytest.mark.parametrize("angles", ["A", "B", "C", "AT", "D"])
@pytest.mark.parametrize("n", [3, 1_001, 300_007])
def test_device_geometry_byte_identical_and_survivors(family, angles, n):
    xy = synth.generate(family, n, seed=n % 97 + 5)
    pts = torch.from_numpy(xy).cuda()
    ws = cp.Workspace(n)
    ext = cp.extremes(pts, angles, ws=ws)                   # K1 leaves its result in ws too
    out_idx, out_pts, count = cp.filter_device(pts, ws=ws)  # Step 2 on the device, then K2
    torch.cuda.synchronize()
    host_geom = cp.geometry(ext)
    host_poly = bytes(cp.polygon(ext).raw)
    dev_geom, dev_poly = _device_pages(ws, len(host_geom))
    assert dev_geom == host_geom
    assert dev_poly == host_poly
    m = int(count.item())
    want = oracle.cudapre(xy, angles, threads=THREADS)
    assert np.array_equal(out_idx[:m].cpu().numpy(), want["survivors"])
    assert np.array_equal(out_pts[:m].cpu().numpy(), xy[want["survivors"]])


def test_device_geometry_adversarial_inputs():
    """Ties, collinear extremes, far-off centres, tiny and huge magnitudes."""
    rng = np.random.default_rng(4)
    cases = [
        np.round(synth.generate("disk", 50_001, seed=1) * 8).astype(np.float32),       # heavy ties
        np.stack([np.linspace(-1, 1, 20_001), np.linspace(-1, 1, 20_001) * 0.5], 1).astype(np.float32),
        (synth.generate("disk", 80_001, seed=2) + np.float32(4096.0)).astype(np.float32),
        (synth.generate("gauss", 80_001, seed=3).astype(np.float64) * 1e-30).astype(np.float32),
        (synth.generate("square", 80_001, seed=4).astype(np.float64) * 1e30).astype(np.float32),
        rng.integers(-3, 4, (60_001, 2)).astype(np.float32),                              # lattice
    ]
    for xy in cases:
        pts = torch.from_numpy(np.ascontiguousarray(xy)).cuda()
        ws = cp.Workspace(len(xy))
        ext = cp.extremes(pts, "A", ws=ws)
        out_idx, _, count = cp.filter_device(pts, ws=ws, return_points=False)
        torch.cuda.synchronize()
        host_geom = cp.geometry(ext)
        dev_geom, dev_poly = _device_pages(ws, len(host_geom))
        assert dev_geom == host_geom
        assert dev_poly == bytes(cp.polygon(ext).raw)
        want = oracle.cudapre(xy, "A", threads=THREADS)["survivors"]
        assert np.array_equal(out_idx[: int(count.item())].cpu().numpy(), want)


def test_pipeline_and_graph_match_oracle():
    for fam, n in (("disk", 1_000_003), ("square", 300_001), ("circle", 200_003)):
        xy = synth.generate(fam, n, seed=11)
        pts = torch.from_numpy(xy).cuda()
        want = oracle.cudapre(xy, "A", threads=THREADS)["survivors"]
        out_idx, out_pts, count = cp.pipeline(pts, "A")
        torch.cuda.synchronize()
        assert np.array_equal(out_idx[: int(count.item())].cpu().numpy(), want)
        g = cp.Graph(pts, "A")
        for _ in range(3):
            g.count.zero_()
            g.launch()
            torch.cuda.synchronize()
            m = int(g.count.item())
            assert np.array_equal(g.out_idx[:m].cpu().numpy(), want)
            assert np.array_equal(g.out_pts[:m].cpu().numpy(), xy[want])
        g.close()


def test_device_path_degenerate_and_misaligned():
    # all points on one line: degenerate ring, everything survives
    t = np.linspace(-1, 1, 10_001, dtype=np.float32)
    xy = np.stack([t, 2 * t], 1)
    out_idx, _, count = cp.pipeline(torch.from_numpy(xy).cuda(), "A", return_points=False)
    torch.cuda.synchronize()
    assert int(count.item()) == len(xy)
    assert np.array_equal(out_idx[: len(xy)].cpu().numpy(), np.arange(len(xy)))
    # 8-byte aligned input: register K2 kernel with the device geometry
    xy = synth.generate("gauss", 300_000, seed=2)
    full = torch.from_numpy(xy).cuda()
    view = full[1:]
    assert view.data_ptr() % 16 == 8
    out_idx, _, count = cp.pipeline(view, "A", index_base=1, return_points=False)
    torch.cuda.synchronize()
    want = oracle.cudapre(xy[1:], "A", threads=THREADS)["survivors"]
    assert np.array_equal(out_idx[: int(count.item())].cpu().numpy() - 1, want)


@pytest.mark.parametrize("k", [2, 3, 8])
def test_device_merge_of_shards(k):
    """The device builder's merge of k per-shard Step-1 blocks (what an NCCL
    all-gather delivers) equals cudapre_extremes_merge + the host polygon,
    byte for byte, and the sharded device pipeline returns the oracle's
    survivors (ties across shard borders included)."""
    xy = np.round(synth.generate("disk", 400_003, seed=17) * 64).astype(np.float32)   # heavy ties
    n = len(xy)
    bounds = [n * r // k for r in range(k + 1)]
    gathered = torch.empty(k * cp.EXTREMES_BYTES, dtype=torch.uint8, device="cuda")
    parts, shards = [], []
    for r in range(k):
        lo, hi = bounds[r], bounds[r + 1]
        pts = torch.from_numpy(np.ascontiguousarray(xy[lo:hi])).cuda()
        ws = cp.Workspace(hi - lo)
        ext = cp.extremes(pts, "A", index_base=lo, ws=ws)      # host copy for the reference merge
        gathered[r * cp.EXTREMES_BYTES:(r + 1) * cp.EXTREMES_BYTES].copy_(cp.result_view(ws))
        parts.append(ext.raw)
        shards.append((pts, ws, lo))
    merged = cp.merge(parts)
    want = oracle.cudapre(xy, "A", threads=THREADS)["survivors"]
    got = []
    for pts, ws, lo in shards:
        cp.polygon_device(ws, parts=gathered, nparts=k)
        out_idx = torch.empty(pts.shape[0], dtype=torch.int64, device="cuda")
        count = torch.zeros(1, dtype=torch.int64, device="cuda")
        cp.filter_geom(pts, index_base=lo, ws=ws, out_idx=out_idx, count=count)
        torch.cuda.synchronize()
        host_geom = cp.geometry(merged)
        dev_geom, dev_poly = _device_pages(ws, len(host_geom))
        assert dev_geom == host_geom
        assert dev_poly == bytes(cp.polygon(merged).raw)
        assert bytes(cp.result_view(ws).cpu().numpy().tobytes()) == bytes(merged.raw)
        got.append(out_idx[: int(count.item())].cpu().numpy())
    assert np.array_equal(np.concatenate(got), want)


@pytest.mark.parametrize("n", [1, 2, 4, 7])
def test_device_path_tiny_inputs(n):
    xy = synth.generate("disk", n, seed=n + 40)
    pts = torch.from_numpy(xy).cuda()
    want = oracle.cudapre(xy, "A", threads=1)["survivors"]
    out_idx, out_pts, count = cp.pipeline(pts, "A")
    torch.cuda.synchronize()
    m = int(count.item())
    assert np.array_equal(out_idx[:m].cpu().numpy(), want)
    g = cp.Graph(pts, "A")
    g.launch()
    torch.cuda.synchronize()
    assert np.array_equal(g.out_idx[: int(g.count.item())].cpu().numpy(), want)
    g.close()


def test_device_path_single_repeated_point_and_empty():
    xy = np.tile(np.array([[0.25, -0.5]], np.float32), (70_000, 1))   # one distinct point
    out_idx, _, count = cp.pipeline(torch.from_numpy(xy).cuda(), "A", return_points=False)
    torch.cuda.synchronize()
    assert int(count.item()) == len(xy)                                # degenerate ring: all kept
    with pytest.raises(cp.CudaPreError) as e:
        cp.pipeline(torch.empty((0, 2), device="cuda"), "A")
    assert e.value.status == cp.ERR_EMPTY


@pytest.mark.parametrize("family", ["square", "disk", "gauss", "circle"])
@pytest.mark.parametrize("angles", ["A", "D"])
def test_pipeline_host_matches_oracle(family, angles):
    """cudapre_pipeline_host — the paper's host Step 2 between the kernels in
    one call (K1 writes the picks into mapped host memory): survivors,
    coordinates and the polygon equal the oracle's, for 16- and 8-byte
    aligned input (TMA and register kernels), ragged sizes and an
    index_base."""
    for n, base, misalign in ((1_000_003, 0, False), (65_537, 7_000_000_000, False), (300_007, 0, True), (5, 0, False)):
        xy = synth.generate(family, n, seed=21)
        want = oracle.cudapre(xy, angles, threads=THREADS)
        if misalign:
            buf = torch.empty((n + 1, 2), dtype=torch.float32, device="cuda")
            buf[1:] = torch.from_numpy(xy).cuda()
            pts = buf[1:]
        else:
            pts = torch.from_numpy(xy).cuda()
        polys = []
        out_idx, out_pts, count = cp.pipeline_host(pts, angles, index_base=base, polygon_out=polys)
        torch.cuda.synchronize()
        m = int(count.item())
        got = out_idx[:m].cpu().numpy()
        assert np.array_equal(got - base, want["survivors"]), (family, angles, n)
        assert np.array_equal(out_pts[:m].cpu().numpy(), xy[want["survivors"]])
        poly = polys[0][0]
        assert poly.degenerate == want["degenerate"]
        if not want["degenerate"]:
            assert (poly.vidx - base).tolist() == want["ring"].tolist()


def test_pipeline_host_alternating_streams():
    """Back-to-back pipeline_host calls on two streams and two inputs (the
    per-thread staging buffer is reused: a call waits for the previous
    call's geometry copy before overwriting it) give each input its own
    oracle survivors."""
    xa = synth.generate("disk", 2_000_003, seed=31)
    xb = synth.generate("square", 1_500_001, seed=32)
    wa = oracle.cudapre(xa, "A", threads=THREADS)["survivors"]
    wb = oracle.cudapre(xb, "A", threads=THREADS)["survivors"]
    pa, pb = torch.from_numpy(xa).cuda(), torch.from_numpy(xb).cuda()
    wsa, wsb = cp.Workspace(len(xa)), cp.Workspace(len(xb))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(4):
        ia, _, ca = cp.pipeline_host(pa, "A", ws=wsa, stream=s1, return_points=False)
        ib, _, cb = cp.pipeline_host(pb, "A", ws=wsb, stream=s2, return_points=False)
        torch.cuda.synchronize()
        assert np.array_equal(ia[: int(ca.item())].cpu().numpy(), wa)
        assert np.array_equal(ib[: int(cb.item())].cpu().numpy(), wb)
