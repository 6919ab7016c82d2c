"""B200-native CudaPre interior-point filter (G. Mei, arXiv 1405.3454).

Thin ctypes binding over ``libcudapre.so`` (include/cudapre.h).  This module
only marshals arguments: every step of the hot path runs in the library's
CUDA kernels (Step 1, Step 3) and host C++ (Step 2, final hull).  PyTorch
supplies device memory, streams and process groups.  There is no CPU
fallback: importing works anywhere, but any compute call raises if the
library or a CUDA device is missing.

    pts = torch.as_tensor(xy, device="cuda")           # (n, 2) float32
    ext = cudapre.extremes(pts)                        # Step 1
    idx, surv, rep = cudapre.filter(pts, ext)          # Steps 2+3
    ring = cudapre.hull(surv.cpu().numpy())            # final hull

Multi-GPU (one process per GPU, torch.distributed over NCCL): each rank
passes its shard and ``index_base``; ``extremes(..., group=pg)`` all-gathers
the per-rank results (one 912-byte struct per rank) and merges them with the
library's lexicographic rule, so every rank gets the single-GPU answer.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcudapre.so")
MAX_ANGLES = 8
MAX_SLOTS = 32
SECTORS = 1024

OK, ERR_EMPTY, ERR_ARG, ERR_NONFINITE, ERR_CUDA, ERR_CAPACITY, ERR_WORKSPACE, ERR_NCCL = range(8)
_STATUS = {1: "EMPTY_INPUT", 2: "INVALID_ARGUMENT", 3: "NONFINITE_INPUT", 4: "CUDA",
           5: "CAPACITY", 6: "WORKSPACE", 7: "NCCL"}
PRESETS = {"A": 0, "B": 1, "AT": 2, "C": 3, "D": 4}   # {0,30,45,60} {0,30,45,45} {0} {0,22.5,45,67.5} {0,15,..,75}


class CudaPreError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"cudapre {_STATUS.get(status, status)}: {msg}")
        self.status = status


class Pt(ctypes.Structure):
    _fields_ = [("x", ctypes.c_float), ("y", ctypes.c_float)]


class ExtremesT(ctypes.Structure):
    _fields_ = [("nang", ctypes.c_int32), ("nonfinite", ctypes.c_int32), ("n", ctypes.c_int64),
                ("idx", ctypes.c_int64 * MAX_SLOTS), ("key", ctypes.c_double * MAX_SLOTS),
                ("pt", Pt * MAX_SLOTS), ("c", ctypes.c_double * MAX_ANGLES),
                ("s", ctypes.c_double * MAX_ANGLES), ("exact_points", ctypes.c_int64)]


class PolygonT(ctypes.Structure):
    _fields_ = [("nv", ctypes.c_int32), ("degenerate", ctypes.c_int32),
                ("n_distinct", ctypes.c_int32), ("exact_only", ctypes.c_int32),
                ("vidx", ctypes.c_int64 * MAX_SLOTS), ("v", Pt * MAX_SLOTS),
                ("box", ctypes.c_float * 4), ("circle", ctypes.c_float * 4),
                ("err_max", ctypes.c_float), ("pad", ctypes.c_int32),
                ("A", ctypes.c_float * MAX_SLOTS), ("B", ctypes.c_float * MAX_SLOTS),
                ("C", ctypes.c_float * MAX_SLOTS), ("E", ctypes.c_float * MAX_SLOTS),
                ("sector_r2", ctypes.c_float * (SECTORS + 1)),
                ("sector_out_r2", ctypes.c_float * (SECTORS + 1))]


class ReportT(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("survivors", ctypes.c_int64),
                ("ms_extremes_kernels", ctypes.c_double), ("ms_filter_kernel", ctypes.c_double),
                ("ms_polygon_host", ctypes.c_double), ("launches", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("lookback_rounds", ctypes.c_int64),
                ("lookback_spins", ctypes.c_int64)]


EXTREMES_BYTES = ctypes.sizeof(ExtremesT)

MAX_SLOTS3 = 6 * 8     # CUDAPRE3_MAX_SLOTS
MAX_FACETS3 = 64       # CUDAPRE3_MAX_FACETS


class Pt3(ctypes.Structure):
    _fields_ = [("x", ctypes.c_float), ("y", ctypes.c_float), ("z", ctypes.c_float)]


class Extremes3T(ctypes.Structure):
    _fields_ = [("nang", ctypes.c_int32), ("nonfinite", ctypes.c_int32), ("n", ctypes.c_int64),
                ("idx", ctypes.c_int64 * MAX_SLOTS3), ("key", ctypes.c_double * MAX_SLOTS3),
                ("pt", Pt3 * MAX_SLOTS3), ("c", ctypes.c_double * 8), ("s", ctypes.c_double * 8),
                ("exact_points", ctypes.c_int64)]


class Polyhedron3T(ctypes.Structure):
    _fields_ = [("nf", ctypes.c_int32), ("n_distinct", ctypes.c_int32), ("cells", ctypes.c_int32),
                ("n_entries", ctypes.c_int32), ("eidx", ctypes.c_int64 * MAX_SLOTS3),
                ("fidx", (ctypes.c_int64 * 3) * MAX_FACETS3), ("fv", (Pt3 * 3) * MAX_FACETS3),
                ("centre", ctypes.c_float * 3), ("err_max", ctypes.c_float),
                ("max_candidates", ctypes.c_int32), ("long_cells", ctypes.c_int32), ("n_cells", ctypes.c_int32),
                ("empty_cells", ctypes.c_int32), ("pad", ctypes.c_int32 * 4)]


SYMBOLS = ["cudapre_version", "cudapre_last_error", "cudapre_angles_preset",
           "cudapre_workspace_bytes", "cudapre_workspace_init", "cudapre_extremes",
           "cudapre_extremes_merge", "cudapre_polygon", "cudapre_filter", "cudapre_hull",
           "cudapre_run_host", "cudapre_geometry", "cudapre_filter_device", "cudapre_pipeline_device",
           "cudapre_graph_create", "cudapre_graph_launch", "cudapre_graph_destroy", "cudapre_pipeline_host",
           "cudapre_polygon_device", "cudapre_filter_geom", "cudapre_hull_device_bytes",
           "cudapre_hull_device", "cudapre_hull_device_ex",
           # multi-GPU (in-library NCCL communicator)
           "cudapre_comm_unique_id", "cudapre_comm_create", "cudapre_comm_destroy", "cudapre_comm_rank",
           "cudapre_comm_allgather_extremes", "cudapre_extremes_comm", "cudapre_pipeline_comm",
           "cudapre_gather_survivors", "cudapre_hull_comm",
           # the 3D extension
           "cudapre3_workspace_bytes", "cudapre3_orient", "cudapre3_extremes", "cudapre3_extremes_merge",
           "cudapre3_polyhedron", "cudapre3_filter", "cudapre3_filter_ex", "cudapre3_cells", "cudapre3_planes"]
WS_GEOM_OFFSET = 4096            # include/cudapre.h CUDAPRE_WS_GEOM_OFFSET
WS_POLY_OFFSET = 4096 + 16384    # CUDAPRE_WS_POLY_OFFSET
WS_RESULT_OFFSET = 176           # CUDAPRE_WS_RESULT_OFFSET

_lib = None


def lib():
    """Load libcudapre.so (built by paper_1405_3454_b200.build); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1405_3454_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    P = ctypes.POINTER
    L.cudapre_version.restype = ctypes.c_char_p
    L.cudapre_last_error.restype = ctypes.c_char_p
    L.cudapre_angles_preset.argtypes = [ctypes.c_int, P(i32), P(ctypes.c_double), P(ctypes.c_double)]
    L.cudapre_workspace_bytes.argtypes = [i64]
    L.cudapre_workspace_bytes.restype = sz
    L.cudapre_workspace_init.argtypes = [vp, sz, vp]
    L.cudapre_extremes.argtypes = [vp, i64, i64, i32, vp, vp, vp, sz, vp, vp, P(ExtremesT), P(ReportT)]
    L.cudapre_extremes_merge.argtypes = [P(ExtremesT), i32, P(ExtremesT)]
    L.cudapre_polygon.argtypes = [P(ExtremesT), P(PolygonT)]
    L.cudapre_filter.argtypes = [vp, i64, i64, P(ExtremesT), vp, vp, i64, vp, sz, vp, P(i64),
                                 P(PolygonT), P(ReportT)]
    L.cudapre_hull.argtypes = [vp, vp, i64, vp, P(i64)]
    L.cudapre_run_host.argtypes = [vp, i64, i32, vp, vp, vp, vp, sz, vp, vp, i64, vp, P(i64), P(ReportT)]
    L.cudapre_geometry.argtypes = [P(ExtremesT), vp, sz, P(sz)]
    L.cudapre_filter_device.argtypes = [vp, i64, i64, vp, vp, vp, i64, vp, sz, vp, vp, vp]
    L.cudapre_pipeline_device.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp, i64, vp, sz, vp, vp]
    L.cudapre_pipeline_host.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp, i64, vp, sz, vp, vp, P(PolygonT),
                                         P(ctypes.c_double)]
    L.cudapre_graph_create.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp, i64, vp, sz, vp, vp, P(vp)]
    L.cudapre_graph_launch.argtypes = [vp, vp]
    L.cudapre_graph_destroy.argtypes = [vp]
    L.cudapre_polygon_device.argtypes = [vp, i32, vp, sz, vp, vp]
    L.cudapre_filter_geom.argtypes = [vp, i64, i64, vp, vp, i64, vp, sz, vp, vp]
    L.cudapre_hull_device_bytes.argtypes = [i64]
    L.cudapre_hull_device_bytes.restype = sz
    L.cudapre_hull_device.argtypes = [vp, vp, i64, P(PolygonT), vp, sz, vp, vp, i64, P(i64), P(i64)]
    L.cudapre_hull_device_ex.argtypes = [vp, vp, i64, P(PolygonT), vp, sz, vp, vp, vp, i64, P(i64), P(i64)]
    L.cudapre_comm_unique_id.argtypes = [vp]
    L.cudapre_comm_create.argtypes = [vp, i32, i32, P(vp)]
    L.cudapre_comm_destroy.argtypes = [vp]
    L.cudapre_comm_rank.argtypes = [vp, P(i32), P(i32)]
    L.cudapre_comm_allgather_extremes.argtypes = [vp, vp, vp, vp]
    L.cudapre_extremes_comm.argtypes = [vp, i64, i64, i32, vp, vp, vp, sz, vp, vp, vp, P(ExtremesT)]
    L.cudapre_pipeline_comm.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp, i64, vp, sz, vp, vp, vp, vp]
    L.cudapre_gather_survivors.argtypes = [vp, vp, vp, i64, i32, vp, vp, i64, vp, P(i64)]
    L.cudapre_hull_comm.argtypes = [vp, vp, vp, i64, P(PolygonT), vp, sz, i32, vp, vp, i64, P(i64)]
    L.cudapre3_workspace_bytes.argtypes = [i64]
    L.cudapre3_workspace_bytes.restype = sz
    L.cudapre3_orient.argtypes = [vp, vp, vp, vp]
    L.cudapre3_extremes.argtypes = [vp, i64, i64, i32, vp, vp, vp, sz, vp, vp, P(Extremes3T), vp]
    L.cudapre3_extremes_merge.argtypes = [P(Extremes3T), i32, P(Extremes3T)]
    L.cudapre3_polyhedron.argtypes = [P(Extremes3T), P(Polyhedron3T)]
    L.cudapre3_cells.argtypes = [P(Extremes3T), vp, i32, vp, P(i32), P(i32)]
    L.cudapre3_planes.argtypes = [P(Extremes3T), vp, i32, P(i32)]
    L.cudapre3_filter.argtypes = [vp, i64, i64, P(Extremes3T), vp, vp, i64, vp, sz, vp, P(i64), P(Polyhedron3T), vp]
    L.cudapre3_filter_ex.argtypes = [vp, i64, i64, P(Extremes3T), vp, vp, i64, vp, sz, vp, P(i64), P(Polyhedron3T), vp,
                                     i32]
    for name in SYMBOLS[2:]:
        if name not in ("cudapre_workspace_bytes", "cudapre_hull_device_bytes", "cudapre3_workspace_bytes"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(status: int, allow=()):
    if status != OK and status not in allow:
        raise CudaPreError(status, lib().cudapre_last_error().decode())
    return status


# ------------------------------------------------------------------ angles
def angles(preset="A"):
    """(nang, c[8], s[8]) of a preset — correctly rounded coefficients (A5)."""
    n = ctypes.c_int32()
    c = (ctypes.c_double * MAX_ANGLES)()
    s = (ctypes.c_double * MAX_ANGLES)()
    _check(lib().cudapre_angles_preset(PRESETS.get(preset, preset), ctypes.byref(n), c, s))
    return n.value, np.frombuffer(c, np.float64).copy(), np.frombuffer(s, np.float64).copy()


# ------------------------------------------------------------------ torch plumbing
def _torch():
    import torch

    return torch


def _stream_ptr(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _points(pts):
    torch = _torch()
    if not isinstance(pts, torch.Tensor) or not pts.is_cuda:
        raise TypeError("points must be a CUDA tensor of shape (n, 2), float32")
    if pts.dtype != torch.float32 or pts.dim() != 2 or pts.shape[1] != 2 or not pts.is_contiguous():
        raise TypeError("points must be a contiguous (n, 2) float32 tensor")
    return pts


class Workspace:
    """Caller-owned device workspace (a zero-filled uint8 tensor)."""

    def __init__(self, n_local: int, device=None):
        torch = _torch()
        self.nbytes = int(lib().cudapre_workspace_bytes(int(n_local)))
        self.capacity_points = int(n_local)
        self.tensor = torch.zeros(self.nbytes, dtype=torch.uint8, device=device or "cuda")

    @property
    def ptr(self):
        return ctypes.c_void_p(self.tensor.data_ptr())


_ws_cache: dict = {}


def _workspace(n: int, device, ws):
    if ws is not None:
        return ws
    torch = _torch()
    dev = torch.device(device)
    key = (dev.index if dev.index is not None else torch.cuda.current_device())
    cur = _ws_cache.get(key)
    if cur is None or cur.capacity_points < n:
        cur = Workspace(max(n, 1), device=dev)
        _ws_cache[key] = cur
    return cur


@dataclass
class Extremes:
    """Step-1 result (slot 4k+{argmin X, argmax X, argmin Y, argmax Y})."""
    raw: ExtremesT

    @property
    def nang(self):
        return self.raw.nang

    @property
    def n(self):
        return self.raw.n

    @property
    def idx(self) -> np.ndarray:
        return np.frombuffer(self.raw.idx, np.int64)[: 4 * self.nang].copy()

    @property
    def key(self) -> np.ndarray:
        return np.frombuffer(self.raw.key, np.float64)[: 4 * self.nang].copy()

    @property
    def pt(self) -> np.ndarray:
        return np.frombuffer(self.raw.pt, np.float32).reshape(-1, 2)[: 4 * self.nang].copy()


@dataclass
class Polygon:
    raw: PolygonT

    @property
    def nv(self):
        return self.raw.nv

    @property
    def degenerate(self):
        return bool(self.raw.degenerate)

    @property
    def vidx(self) -> np.ndarray:
        return np.frombuffer(self.raw.vidx, np.int64)[: self.nv].copy()

    @property
    def v(self) -> np.ndarray:
        return np.frombuffer(self.raw.v, np.float32).reshape(-1, 2)[: self.nv].copy()

    @property
    def box(self):
        return tuple(self.raw.box)

    @property
    def circle(self):
        return tuple(self.raw.circle[:3])


def _angle_arrays(angle_set):
    if isinstance(angle_set, (str, int)):
        return angles(angle_set)
    c, s = angle_set
    c = np.asarray(c, np.float64)
    s = np.asarray(s, np.float64)
    cc = np.zeros(MAX_ANGLES)
    ss = np.zeros(MAX_ANGLES)
    cc[: len(c)] = c
    ss[: len(s)] = s
    return len(c), cc, ss


# ------------------------------------------------------------------ Step 1
def extremes(pts, angles_="A", index_base: int = 0, group=None, ws=None, stream=None,
             report: ReportT | None = None, device_out=None) -> Extremes:
    """Step 1 on the local shard; with ``group`` the
    per-rank results are all-gathered (torch.distributed) and merged."""
    torch = _torch()
    pts = _points(pts)
    n = pts.shape[0]
    nang, c, s = _angle_arrays(angles_)
    w = _workspace(n, pts.device, ws)
    out = ExtremesT()
    on_device = False
    if group is not None:
        import torch.distributed as dist

        on_device = dist.get_backend(group) == "nccl"
    dev_buf = device_out
    if on_device and dev_buf is None:
        dev_buf = torch.empty(EXTREMES_BYTES, dtype=torch.uint8, device=pts.device)
    want_host = not on_device
    st = lib().cudapre_extremes(
        ctypes.c_void_p(pts.data_ptr()), n, index_base, nang,
        c.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p),
        w.ptr, w.nbytes, _stream_ptr(stream),
        ctypes.c_void_p(dev_buf.data_ptr()) if dev_buf is not None else None,
        ctypes.byref(out) if want_host else None,
        ctypes.byref(report) if report is not None else None)
    if group is None:
        _check(st)
        return Extremes(out)
    _check(st, allow=(ERR_EMPTY, ERR_NONFINITE))
    return exchange(out, group, dev_buf if on_device else None)


def exchange(local: ExtremesT, group, device_buf=None) -> Extremes:
    """Cross-rank combine: all-gather every rank's Step-1
    struct (NCCL: straight from the device buffer K1 wrote; gloo: host bytes)
    and merge them with the library's lexicographic rule."""
    torch = _torch()
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if device_buf is not None:
        gathered = torch.empty(world * EXTREMES_BYTES, dtype=torch.uint8, device=device_buf.device)
        dist.all_gather_into_tensor(gathered, device_buf, group=group)
        host = gathered.cpu().numpy().tobytes()
    else:
        mine = torch.frombuffer(bytearray(bytes(local)), dtype=torch.uint8)
        bufs = [torch.empty(EXTREMES_BYTES, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(bufs, mine, group=group)
        host = b"".join(bytes(b.numpy().tobytes()) for b in bufs)
    parts = (ExtremesT * world).from_buffer_copy(host)
    return merge(list(parts))


def merge(parts) -> Extremes:
    """Combine per-shard Step-1 results."""
    arr = (ExtremesT * len(parts))(*[p.raw if isinstance(p, Extremes) else p for p in parts])
    out = ExtremesT()
    _check(lib().cudapre_extremes_merge(arr, len(parts), ctypes.byref(out)))
    return Extremes(out)


# ------------------------------------------------------------------ Step 2
def polygon(ext: Extremes) -> Polygon:
    out = PolygonT()
    _check(lib().cudapre_polygon(ctypes.byref(ext.raw), ctypes.byref(out)))
    return Polygon(out)


# ------------------------------------------------------------------ Step 3
def filter(pts, ext: Extremes, index_base: int = 0, return_points: bool = True, ws=None,
           out_idx=None, out_pts=None, stream=None):
    """Steps 2+3: survivors' global indices (ascending,
    int64 CUDA tensor), optionally their coordinates, and a report dict."""
    torch = _torch()
    pts = _points(pts)
    n = pts.shape[0]
    w = _workspace(n, pts.device, ws)
    if out_idx is None:
        out_idx = torch.empty(max(n, 1), dtype=torch.int64, device=pts.device)
    if return_points and out_pts is None:
        out_pts = torch.empty((max(n, 1), 2), dtype=torch.float32, device=pts.device)
    cap = out_idx.shape[0]
    if out_pts is not None:
        cap = min(cap, out_pts.shape[0])
    count = ctypes.c_int64()
    poly = PolygonT()
    rep = ReportT()
    _check(lib().cudapre_filter(
        ctypes.c_void_p(pts.data_ptr()), n, index_base, ctypes.byref(ext.raw),
        ctypes.c_void_p(out_idx.data_ptr()),
        ctypes.c_void_p(out_pts.data_ptr()) if out_pts is not None else None,
        cap, w.ptr, w.nbytes, _stream_ptr(stream), ctypes.byref(count), ctypes.byref(poly),
        ctypes.byref(rep)))
    m = count.value
    return (out_idx[:m], out_pts[:m] if out_pts is not None else None,
            {"n": n, "survivors": m, "polygon": Polygon(poly),
             "ms_filter_kernel": rep.ms_filter_kernel, "ms_polygon_host": rep.ms_polygon_host,
             "launches": rep.launches, "lookback_rounds": rep.lookback_rounds,
             "lookback_spins": rep.lookback_spins})


# ------------------------------------------------------------------ final hull
def hull(xy, ids=None) -> np.ndarray:
    """Canonical convex-hull ring of host points (numpy
    (n, 2) float32 or CPU tensor), over ``ids`` if given."""
    p = np.ascontiguousarray(np.asarray(xy, np.float32).reshape(-1, 2))
    if ids is None:
        m = len(p)
        ids_a = None
    else:
        ids_a = np.ascontiguousarray(np.asarray(ids, np.int64))
        m = len(ids_a)
    ring = np.empty(max(m, 1), np.int64)
    k = ctypes.c_int64()
    _check(lib().cudapre_hull(p.ctypes.data_as(ctypes.c_void_p),
                              None if ids_a is None else ids_a.ctypes.data_as(ctypes.c_void_p),
                              m, ring.ctypes.data_as(ctypes.c_void_p), ctypes.byref(k)))
    return ring[: k.value].copy()


# ------------------------------------------------------------------ whole method
# ------------------------------------------------------------------ device-resident Steps 2-3 (f3)
def geometry(ext: Extremes) -> bytes:
    """Host build of the Step-3 geometry block (the bytes the device builder
    writes at WS_GEOM_OFFSET of the workspace)."""
    need = ctypes.c_size_t()
    lib().cudapre_geometry(ctypes.byref(ext.raw), None, 0, ctypes.byref(need))
    buf = (ctypes.c_uint8 * need.value)()
    _check(lib().cudapre_geometry(ctypes.byref(ext.raw), buf, need.value, None))
    return bytes(buf)


def _outputs(pts, out_idx, out_pts, return_points):
    torch = _torch()
    n = pts.shape[0]
    if out_idx is None:
        out_idx = torch.empty(max(n, 1), dtype=torch.int64, device=pts.device)
    if return_points and out_pts is None:
        out_pts = torch.empty((max(n, 1), 2), dtype=torch.float32, device=pts.device)
    cap = out_idx.shape[0] if out_pts is None else min(out_idx.shape[0], out_pts.shape[0])
    return out_idx, out_pts, cap


def filter_device(pts, ext_dev=None, index_base: int = 0, return_points: bool = True, ws=None,
                  out_idx=None, out_pts=None, d_poly=None, stream=None):
    """Steps 2+3 with Step 2 on the device (no host round trip): returns
    (out_idx, out_pts, count) where count is a device int64 tensor of one
    element (the survivors are out_idx[:count]).  ext_dev: device
    cudapre_extremes_t bytes (None: the result extremes() left in ws)."""
    torch = _torch()
    pts = _points(pts)
    n = pts.shape[0]
    w = _workspace(n, pts.device, ws)
    out_idx, out_pts, cap = _outputs(pts, out_idx, out_pts, return_points)
    count = torch.zeros(1, dtype=torch.int64, device=pts.device)
    _check(lib().cudapre_filter_device(
        ctypes.c_void_p(pts.data_ptr()), n, index_base,
        ctypes.c_void_p(ext_dev.data_ptr()) if ext_dev is not None else None,
        ctypes.c_void_p(out_idx.data_ptr()),
        ctypes.c_void_p(out_pts.data_ptr()) if out_pts is not None else None, cap,
        w.ptr, w.nbytes, _stream_ptr(stream), ctypes.c_void_p(count.data_ptr()),
        ctypes.c_void_p(d_poly.data_ptr()) if d_poly is not None else None))
    return out_idx, out_pts, count


def extremes_device(pts, angles_="A", index_base: int = 0, ws=None, stream=None):
    """Step 1 with no host output and no synchronisation: the result stays in
    the workspace for polygon_device / filter_device."""
    pts = _points(pts)
    n = pts.shape[0]
    nang, c, s = _angle_arrays(angles_)
    w = _workspace(n, pts.device, ws)
    _check(lib().cudapre_extremes(
        ctypes.c_void_p(pts.data_ptr()), n, index_base, nang,
        c.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p),
        w.ptr, w.nbytes, _stream_ptr(stream), None, None, None))


def polygon_device(ws, parts=None, nparts: int = 0, d_poly=None, stream=None):
    """Step 2 on the device into the workspace pages.  parts: a device buffer
    of nparts Step-1 results (EXTREMES_BYTES each, e.g. an all-gather of every
    rank's result_view(ws)), merged first; None: the result in ws."""
    _check(lib().cudapre_polygon_device(
        ctypes.c_void_p(parts.data_ptr()) if parts is not None else None, int(nparts), ws.ptr, ws.nbytes,
        _stream_ptr(stream), ctypes.c_void_p(d_poly.data_ptr()) if d_poly is not None else None))


def result_view(ws):
    """The workspace's Step-1 result block as a uint8 device tensor (no copy)."""
    return ws.tensor[WS_RESULT_OFFSET:WS_RESULT_OFFSET + EXTREMES_BYTES]


def filter_geom(pts, index_base: int = 0, ws=None, out_idx=None, out_pts=None, count=None, stream=None):
    """Step 3 alone on the geometry already in ws; count: device int64[1]."""
    pts = _points(pts)
    n = pts.shape[0]
    w = _workspace(n, pts.device, ws)
    cap = out_idx.shape[0] if out_pts is None else min(out_idx.shape[0], out_pts.shape[0])
    _check(lib().cudapre_filter_geom(
        ctypes.c_void_p(pts.data_ptr()), n, index_base, ctypes.c_void_p(out_idx.data_ptr()),
        ctypes.c_void_p(out_pts.data_ptr()) if out_pts is not None else None, cap, w.ptr, w.nbytes,
        _stream_ptr(stream), ctypes.c_void_p(count.data_ptr()) if count is not None else None))


def pipeline(pts, angles_="A", index_base: int = 0, return_points: bool = True, ws=None, out_idx=None,
             out_pts=None, stream=None):
    """Steps 1-3 enqueued on the stream with no host synchronisation; returns
    (out_idx, out_pts, count) as filter_device."""
    torch = _torch()
    pts = _points(pts)
    n = pts.shape[0]
    nang, c, s = _angle_arrays(angles_)
    w = _workspace(n, pts.device, ws)
    out_idx, out_pts, cap = _outputs(pts, out_idx, out_pts, return_points)
    count = torch.zeros(1, dtype=torch.int64, device=pts.device)
    _check(lib().cudapre_pipeline_device(
        ctypes.c_void_p(pts.data_ptr()), n, index_base, nang,
        c.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p),
        ctypes.c_void_p(out_idx.data_ptr()),
        ctypes.c_void_p(out_pts.data_ptr()) if out_pts is not None else None, cap,
        w.ptr, w.nbytes, _stream_ptr(stream), ctypes.c_void_p(count.data_ptr())))
    return out_idx, out_pts, count


def pipeline_host(pts, angles_="A", index_base: int = 0, return_points: bool = True, ws=None, out_idx=None,
                  out_pts=None, stream=None, polygon_out: list | None = None):
    """Steps 1-3 with the paper's host Step 2 between the kernels in one
    library call (cudapre_pipeline_host): one host wait per step, for the
    Step-1 picks; returns (out_idx, out_pts, count) as pipeline().
    ``polygon_out``: a list the Polygon and the host Step-2 ms are appended to."""
    torch = _torch()
    pts = _points(pts)
    n = pts.shape[0]
    nang, c, s = _angle_arrays(angles_)
    w = _workspace(n, pts.device, ws)
    out_idx, out_pts, cap = _outputs(pts, out_idx, out_pts, return_points)
    count = torch.zeros(1, dtype=torch.int64, device=pts.device)
    poly = PolygonT()
    ms = ctypes.c_double()
    _check(lib().cudapre_pipeline_host(
        ctypes.c_void_p(pts.data_ptr()), n, index_base, nang,
        c.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p),
        ctypes.c_void_p(out_idx.data_ptr()),
        ctypes.c_void_p(out_pts.data_ptr()) if out_pts is not None else None, cap,
        w.ptr, w.nbytes, _stream_ptr(stream), ctypes.c_void_p(count.data_ptr()), ctypes.byref(poly),
        ctypes.byref(ms)))
    if polygon_out is not None:
        polygon_out.append((Polygon(poly), ms.value))
    return out_idx, out_pts, count


class Graph:
    """Steps 1-3 captured once in a CUDA graph on fixed buffers; launch()
    replays the whole step with one graph launch.  count is a device int64
    tensor updated by every launch."""

    def __init__(self, pts, angles_="A", index_base: int = 0, return_points: bool = True, ws=None,
                 out_idx=None, out_pts=None, stream=None):
        torch = _torch()
        self.pts = _points(pts)
        n = self.pts.shape[0]
        nang, c, s = _angle_arrays(angles_)
        self.ws = _workspace(n, self.pts.device, ws)
        self.out_idx, self.out_pts, cap = _outputs(self.pts, out_idx, out_pts, return_points)
        self.count = torch.zeros(1, dtype=torch.int64, device=self.pts.device)
        h = ctypes.c_void_p()
        _check(lib().cudapre_graph_create(
            ctypes.c_void_p(self.pts.data_ptr()), n, index_base, nang,
            c.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p),
            ctypes.c_void_p(self.out_idx.data_ptr()),
            ctypes.c_void_p(self.out_pts.data_ptr()) if self.out_pts is not None else None, cap,
            self.ws.ptr, self.ws.nbytes, _stream_ptr(stream), ctypes.c_void_p(self.count.data_ptr()),
            ctypes.byref(h)))
        self._h = h

    def launch(self, stream=None):
        _check(lib().cudapre_graph_launch(self._h, _stream_ptr(stream)))

    def close(self):
        if self._h:
            lib().cudapre_graph_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hull_device(pts, ids, m: int, poly, stream=None, return_remaining: bool = False):
    """Final hull of the survivors pts[:m] (device float2) with
    global ids ids[:m] (device int64), filtered with polygon `poly` (the
    Polygon Step 2 returned): the canonical ring of global ids (numpy)."""
    torch = _torch()
    m = int(m)
    nbytes = int(lib().cudapre_hull_device_bytes(m))
    scratch = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=pts.device)
    ring = np.empty(max(m, 1), np.int64)
    n_ring, rem = ctypes.c_int64(), ctypes.c_int64()
    raw = poly.raw if isinstance(poly, Polygon) else poly
    _check(lib().cudapre_hull_device(
        ctypes.c_void_p(pts.data_ptr()), ctypes.c_void_p(ids.data_ptr()), m, ctypes.byref(raw),
        ctypes.c_void_p(scratch.data_ptr()), nbytes, _stream_ptr(stream),
        ring.ctypes.data_as(ctypes.c_void_p), len(ring), ctypes.byref(n_ring), ctypes.byref(rem)))
    out = ring[: n_ring.value].copy()
    return (out, rem.value) if return_remaining else out


# ------------------------------------------------------------------ multi-GPU (in-library NCCL)
class Comm:
    """In-library NCCL communicator (cudapre_comm_*), one per process/GPU,
    bound to the current CUDA device.  ``Comm.from_group(group)`` makes the
    NCCL id on rank 0 and distributes it with torch.distributed (any backend:
    plumbing only)."""

    def __init__(self, rank: int, world: int, unique_id: bytes):
        if len(unique_id) != 128:
            raise ValueError("the NCCL unique id is 128 bytes")
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(unique_id, 128)
        _check(lib().cudapre_comm_create(buf, int(rank), int(world), ctypes.byref(h)))
        self._h, self.rank, self.world = h, int(rank), int(world)

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().cudapre_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_group(cls, group=None):
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        return cls(rank, world, obj[0])

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().cudapre_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def allgather_extremes(comm: Comm, ws, parts, stream=None):
    """NCCL all-gather of every rank's Step-1 result block (the one
    extremes_device left in ``ws``) into ``parts`` (device uint8,
    world * EXTREMES_BYTES), on the stream; merge with polygon_device."""
    _check(lib().cudapre_comm_allgather_extremes(comm.handle, ws.ptr, ctypes.c_void_p(parts.data_ptr()),
                                                 _stream_ptr(stream)))


def extremes_comm(pts, comm: Comm, angles_="A", index_base: int = 0, ws=None, stream=None) -> Extremes:
    """Step 1 of a sharded set (cudapre_extremes_comm): K1 on the local shard,
    NCCL all-gather of the ranks' results, host merge: the single-GPU answer."""
    torch = _torch()
    pts = _points(pts)
    n = pts.shape[0]
    nang, c, s = _angle_arrays(angles_)
    w = _workspace(max(n, 1), pts.device, ws)
    parts = torch.empty(comm.world * EXTREMES_BYTES, dtype=torch.uint8, device=pts.device)
    out = ExtremesT()
    _check(lib().cudapre_extremes_comm(
        ctypes.c_void_p(pts.data_ptr()) if n else None, n, index_base, nang,
        c.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p), w.ptr, w.nbytes,
        comm.handle, ctypes.c_void_p(parts.data_ptr()), _stream_ptr(stream), ctypes.byref(out)))
    return Extremes(out)


def pipeline_comm(pts, comm: Comm, angles_="A", index_base: int = 0, return_points: bool = True, ws=None,
                  out_idx=None, out_pts=None, parts=None, stream=None):
    """Steps 1-3 of a sharded set on the stream (cudapre_pipeline_comm): K1,
    NCCL all-gather, merge + Step 2 on the device, Step 3 on the local shard;
    returns (out_idx, out_pts, count) as filter_device."""
    torch = _torch()
    pts = _points(pts)
    n = pts.shape[0]
    nang, c, s = _angle_arrays(angles_)
    w = _workspace(n, pts.device, ws)
    out_idx, out_pts, cap = _outputs(pts, out_idx, out_pts, return_points)
    if parts is None:
        parts = torch.empty(comm.world * EXTREMES_BYTES, dtype=torch.uint8, device=pts.device)
    count = torch.zeros(1, dtype=torch.int64, device=pts.device)
    _check(lib().cudapre_pipeline_comm(
        ctypes.c_void_p(pts.data_ptr()), n, index_base, nang,
        c.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p),
        ctypes.c_void_p(out_idx.data_ptr()),
        ctypes.c_void_p(out_pts.data_ptr()) if out_pts is not None else None, cap,
        w.ptr, w.nbytes, comm.handle, ctypes.c_void_p(parts.data_ptr()), _stream_ptr(stream),
        ctypes.c_void_p(count.data_ptr())))
    return out_idx, out_pts, count


def gather_survivors(comm: Comm, idx, pts, count: int, root: int = 0, out_idx=None, out_pts=None, stream=None):
    """Collect every rank's survivors on ``root`` in rank order (= ascending
    global index: the single-GPU array).  Returns (idx, pts, total) on the
    root, (None, None, total) elsewhere.  Collective: every rank calls it."""
    torch = _torch()
    h_total = ctypes.c_int64()
    is_root = comm.rank == root
    cap = out_idx.shape[0] if (is_root and out_idx is not None) else 0
    for attempt in range(2):
        st = lib().cudapre_gather_survivors(
            comm.handle, ctypes.c_void_p(idx.data_ptr()),
            ctypes.c_void_p(pts.data_ptr()) if pts is not None else None, int(count), int(root),
            ctypes.c_void_p(out_idx.data_ptr()) if (is_root and out_idx is not None) else None,
            ctypes.c_void_p(out_pts.data_ptr()) if (is_root and out_pts is not None) else None,
            cap, _stream_ptr(stream), ctypes.byref(h_total))
        if st == ERR_CAPACITY and attempt == 0:   # (every rank sees it) size the root's buffers, retry
            if is_root:
                cap = h_total.value
                out_idx = torch.empty(max(cap, 1), dtype=torch.int64, device=idx.device)
                out_pts = (torch.empty((max(cap, 1), 2), dtype=torch.float32, device=idx.device)
                           if pts is not None else None)
            continue
        _check(st)
        break
    m = h_total.value
    if not is_root:
        return None, None, m
    if m == 0:
        return idx[:0], (pts[:0] if pts is not None else None), 0
    return out_idx[:m], (out_pts[:m] if out_pts is not None else None), m


def hull_comm(comm: Comm, pts, ids, m: int, poly, root: int = 0, stream=None) -> np.ndarray:
    """Final hull of a sharded set (cudapre_hull_comm): per-rank GPU hulls of
    the local survivors, their vertices gathered on the root, one chain
    there.  The canonical ring (global ids) on the root, empty elsewhere."""
    torch = _torch()
    m = int(m)
    nbytes = int(lib().cudapre_hull_device_bytes(m))
    scratch = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=pts.device)
    cap = max(m, 1) * comm.world + 64
    ring = np.empty(cap, np.int64)
    k = ctypes.c_int64()
    raw = poly.raw if isinstance(poly, Polygon) else poly
    _check(lib().cudapre_hull_comm(
        comm.handle, ctypes.c_void_p(pts.data_ptr()), ctypes.c_void_p(ids.data_ptr()), m, ctypes.byref(raw),
        ctypes.c_void_p(scratch.data_ptr()), nbytes, int(root), _stream_ptr(stream),
        ring.ctypes.data_as(ctypes.c_void_p), cap, ctypes.byref(k)))
    return ring[: k.value].copy()


def cuda_pre(pts, angles_="A", group=None, index_base: int = 0, return_points=True, ws=None):
    """Steps 1-3.  Empty input: survivors = input, filter skipped."""
    torch = _torch()
    pts = _points(pts)
    if group is None and pts.shape[0] == 0:
        e = torch.empty(0, dtype=torch.int64, device=pts.device)
        return e, pts[:0], {"n": 0, "survivors": 0, "skipped": True}
    ext = extremes(pts, angles_, index_base=index_base, group=group, ws=ws)
    idx, sp, rep = filter(pts, ext, index_base=index_base, return_points=return_points, ws=ws)
    rep["extremes"] = ext
    rep["skipped"] = rep["polygon"].degenerate
    return idx, sp, rep


def run_host(h_pts: np.ndarray, d_pts, d_surv_idx, h_surv_idx: np.ndarray, angles_="A", ws=None,
             stream=None):
    """End to end from host memory through the C ABI (cudapre_run_host)."""
    n = len(h_pts)
    nang, c, s = _angle_arrays(angles_)
    w = _workspace(n, d_pts.device, ws)
    count = ctypes.c_int64()
    rep = ReportT()
    hp = h_pts.data_ptr() if hasattr(h_pts, "data_ptr") else h_pts.ctypes.data
    hs = h_surv_idx.data_ptr() if hasattr(h_surv_idx, "data_ptr") else h_surv_idx.ctypes.data
    _check(lib().cudapre_run_host(
        ctypes.c_void_p(hp), n, nang, c.ctypes.data_as(ctypes.c_void_p),
        s.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(d_pts.data_ptr()), w.ptr, w.nbytes,
        ctypes.c_void_p(d_surv_idx.data_ptr()), ctypes.c_void_p(hs), d_surv_idx.shape[0],
        _stream_ptr(stream), ctypes.byref(count), ctypes.byref(rep)))
    return count.value, rep


# ====================================================================== 3D
# The 3D extension: float32 xyz points.

def _points3(pts):
    torch = _torch()
    if not isinstance(pts, torch.Tensor) or not pts.is_cuda:
        raise TypeError("3D points must be a CUDA tensor of shape (n, 3), float32")
    if pts.dtype != torch.float32 or pts.dim() != 2 or pts.shape[1] != 3 or not pts.is_contiguous():
        raise TypeError("3D points must be a contiguous (n, 3) float32 tensor")
    return pts


class Workspace3:
    """Caller-owned device workspace of the 3D path (zero-filled uint8 tensor)."""

    def __init__(self, n_local: int, device=None):
        torch = _torch()
        self.nbytes = int(lib().cudapre3_workspace_bytes(int(n_local)))
        self.capacity_points = int(n_local)
        self.tensor = torch.zeros(self.nbytes, dtype=torch.uint8, device=device or "cuda")

    @property
    def ptr(self):
        return ctypes.c_void_p(self.tensor.data_ptr())


_ws3_cache: dict = {}


def _workspace3(n: int, device, ws):
    if ws is not None:
        return ws
    torch = _torch()
    dev = torch.device(device)
    key = (dev.index if dev.index is not None else torch.cuda.current_device())
    cur = _ws3_cache.get(key)
    if cur is None or cur.capacity_points < n:
        cur = Workspace3(max(n, 1), device=dev)
        _ws3_cache[key] = cur
    return cur


@dataclass
class Extremes3:
    """3D Step-1 result: slot 6k+{minX, maxX, minY, maxY, minZ, maxZ}."""
    raw: Extremes3T

    @property
    def nang(self):
        return self.raw.nang

    @property
    def n(self):
        return self.raw.n

    @property
    def idx(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.raw.idx)[: 6 * self.raw.nang].copy()

    @property
    def key(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.raw.key)[: 6 * self.raw.nang].copy()

    @property
    def pt(self) -> np.ndarray:
        a = np.frombuffer(bytes(self.raw.pt), np.float32).reshape(-1, 3)
        return a[: 6 * self.raw.nang].copy()


@dataclass
class Polyhedron:
    """3D Step-2 result: facet planes of conv(E) (E on the positive side)."""
    raw: Polyhedron3T

    @property
    def nf(self):
        return self.raw.nf

    @property
    def degenerate(self):
        return self.raw.nf == 0

    @property
    def eidx(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.raw.eidx)[: self.raw.n_distinct].copy()

    @property
    def facets(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.raw.fidx).reshape(-1, 3)[: self.raw.nf].copy()


def orient3d(a, b, c, d) -> int:
    """Exact orient3d sign (det[b-a; c-a; d-a]) of float triples, host side."""
    q = [np.ascontiguousarray(np.asarray(v, np.float32).reshape(3)) for v in (a, b, c, d)]
    return int(lib().cudapre3_orient(*[v.ctypes.data_as(ctypes.c_void_p) for v in q]))


def extremes3(pts, angles_="A", index_base: int = 0, ws=None, stream=None, device_out=None,
              timing: list | None = None) -> Extremes3:
    """3D Step 1 (P:115 with P:33-35) on the local shard.  ``timing``: a list
    the K1-3D launch's device milliseconds are appended to."""
    pts = _points3(pts)
    n = pts.shape[0]
    nang, c, s = _angle_arrays(angles_)
    w = _workspace3(n, pts.device, ws)
    out = Extremes3T()
    ms = ctypes.c_double()
    _check(lib().cudapre3_extremes(
        ctypes.c_void_p(pts.data_ptr()), n, index_base, nang,
        c.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p),
        w.ptr, w.nbytes, _stream_ptr(stream),
        ctypes.c_void_p(device_out.data_ptr()) if device_out is not None else None, ctypes.byref(out),
        ctypes.byref(ms) if timing is not None else None))
    if timing is not None:
        timing.append(ms.value)
    return Extremes3(out)


def exchange3(local, group, device_buf=None) -> Extremes3:
    """Cross-rank combine in 3D: all-gather every rank's Step-1 struct (NCCL:
    from the device buffer K1-3D wrote via ``device_out``; gloo: host bytes)
    and merge them with the library's lexicographic rule."""
    torch = _torch()
    import torch.distributed as dist

    raw_local = local.raw if isinstance(local, Extremes3) else local
    nbytes = ctypes.sizeof(Extremes3T)
    world = dist.get_world_size(group)
    if device_buf is not None:
        gathered = torch.empty(world * nbytes, dtype=torch.uint8, device=device_buf.device)
        dist.all_gather_into_tensor(gathered, device_buf, group=group)
        host = gathered.cpu().numpy().tobytes()
    else:
        mine = torch.frombuffer(bytearray(bytes(raw_local)), dtype=torch.uint8)
        bufs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(bufs, mine, group=group)
        host = b"".join(bytes(b.numpy().tobytes()) for b in bufs)
    return merge3([Extremes3T.from_buffer_copy(host[r * nbytes:(r + 1) * nbytes]) for r in range(world)])


def merge3(parts) -> Extremes3:
    arr = (Extremes3T * len(parts))(*[p.raw if isinstance(p, Extremes3) else p for p in parts])
    out = Extremes3T()
    _check(lib().cudapre3_extremes_merge(arr, len(parts), ctypes.byref(out)))
    return Extremes3(out)


def polyhedron3(ext: Extremes3) -> Polyhedron:
    out = Polyhedron3T()
    _check(lib().cudapre3_polyhedron(ctypes.byref(ext.raw), ctypes.byref(out)))
    return Polyhedron(out)


def cells3(ext: Extremes3):
    """Test hook: (masks[6 G^2] uint64, centre[3], G, cells_in_use) of the
    direction cells K2-3D uses for these extremes (cudapre3_cells)."""
    L = lib()
    grid, used = ctypes.c_int32(), ctypes.c_int32()
    _check(L.cudapre3_cells(ctypes.byref(ext.raw), None, 0, None, ctypes.byref(grid), ctypes.byref(used)))
    n = 6 * grid.value * grid.value
    masks = np.zeros(n, np.uint64)
    centre = np.zeros(3, np.float32)
    _check(L.cudapre3_cells(ctypes.byref(ext.raw), masks.ctypes.data_as(ctypes.c_void_p), n,
                            centre.ctypes.data_as(ctypes.c_void_p), ctypes.byref(grid), ctypes.byref(used)))
    return masks, centre, grid.value, bool(used.value)


def planes3(ext: Extremes3) -> np.ndarray:
    """Test hook: K2-3D's float plane tests, (nf, 5) = (A, B, C, D, E) per facet."""
    nf = ctypes.c_int32()
    out = np.zeros((MAX_FACETS3, 5), np.float32)
    _check(lib().cudapre3_planes(ctypes.byref(ext.raw), out.ctypes.data_as(ctypes.c_void_p), MAX_FACETS3,
                                 ctypes.byref(nf)))
    return out[: nf.value].copy()


FLAG3_NO_CELLS = 1   # CUDAPRE3_FLAG_NO_CELLS


def filter3(pts, ext: Extremes3, index_base: int = 0, return_points: bool = True, ws=None,
            out_idx=None, out_pts=None, stream=None, timing: list | None = None, flags: int = 0):
    """3D Steps 2+3: survivors' global indices (ascending, int64 CUDA tensor),
    optionally their xyz, and the polyhedron used.  ``timing``: a list the
    K2-3D launch's device milliseconds are appended to."""
    torch = _torch()
    pts = _points3(pts)
    n = pts.shape[0]
    w = _workspace3(n, pts.device, ws)
    if out_idx is None:
        out_idx = torch.empty(max(n, 1), dtype=torch.int64, device=pts.device)
    if return_points and out_pts is None:
        out_pts = torch.empty((max(n, 1), 3), dtype=torch.float32, device=pts.device)
    cap = out_idx.shape[0]
    if out_pts is not None:
        cap = min(cap, out_pts.shape[0])
    count = ctypes.c_int64()
    poly = Polyhedron3T()
    ms = ctypes.c_double()
    _check(lib().cudapre3_filter_ex(
        ctypes.c_void_p(pts.data_ptr()), n, index_base, ctypes.byref(ext.raw),
        ctypes.c_void_p(out_idx.data_ptr()),
        ctypes.c_void_p(out_pts.data_ptr()) if out_pts is not None else None,
        cap, w.ptr, w.nbytes, _stream_ptr(stream), ctypes.byref(count), ctypes.byref(poly),
        ctypes.byref(ms) if timing is not None else None, int(flags)))
    if timing is not None:
        timing.append(ms.value)
    m = count.value
    return out_idx[:m], (out_pts[:m] if out_pts is not None else None), Polyhedron(poly)


def cuda_pre3(pts, angles_="A", index_base: int = 0, return_points: bool = True, ws=None):
    """The 3D method: Step 1, Step 2 (host), Step 3 on one GPU."""
    ext = extremes3(pts, angles_, index_base=index_base, ws=ws)
    idx, sp, poly = filter3(pts, ext, index_base=index_base, return_points=return_points, ws=ws)
    return idx, sp, {"extremes": ext, "polyhedron": poly}
