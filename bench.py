"""Benchmark: filtered points/s of the CudaPre hot path (Steps 1-3) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]
    python bench.py --config T4      # the 3D extension, synth.CONFIGS3
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

One step = one pass of the whole hot path over the workload resident in HBM:
Step 1 (seed + K1 kernels, D2H of the 16 picks; for N>1 the NCCL all-gather of
the per-rank picks and the host merge), Step 2 (host monotone chain + kernel
parameters), Step 3 (K2 classify + ordered compaction writing each survivor's
int64 index and float2 coordinates into HBM, D2H of the count).  Workload:
BASELINE.json configs[4] ("C5": 2e9 points uniform in the unit disk, seeded
synthetic, sharded contiguously over the N ranks: strong scaling).

Prints ONE JSON line (rank 0).  See DESIGN.md §8 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "filtered points/sec (Gpts/s) and % of HBM roofline at 1/2/4/8 B200; discard %"
K1_BYTES_PER_PT = 8          # K1 reads each float2 once
K2_BYTES_PER_PT = 8          # K2 reads each float2 once ...
K2_BYTES_PER_SURVIVOR = 16   # ... and writes int64 index + float2 point per survivor


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=0, help="override total points")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--angles", default="A")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--align8", action="store_true",
                    help="feed an 8-byte (not 16-byte) aligned view: the register-loading K1 / K2 kernels")
    ap.add_argument("--no-points", action="store_true",
                    help="write only the survivors' indices (perf experiment; not the benchmark workload)")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return None


class ClockSampler:
    """NVML samples of SM clock + throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def result(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def oracle_rate(pts_host: np.ndarray, threads: int, angles: str):
    """Time the oracle (as it stands) on a host sample; returns (pts/s, n)."""
    import oracle

    oracle.build()
    t0 = time.perf_counter()
    oracle.cudapre(pts_host, angles, threads=threads)
    dt = time.perf_counter() - t0
    return len(pts_host) / dt, dt


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def oracle_phases(pts_host: np.ndarray, threads: int, angles: str) -> dict:
    """The oracle's Steps timed one by one on the same bytes:
    extremes (Step 1), polygon (Step 2), filter (Step 3), hull of the
    survivors, in seconds."""
    import oracle

    t0 = time.perf_counter()
    ext = oracle.extremes(pts_host, angles, threads=threads)
    t1 = time.perf_counter()
    ring = oracle.polygon(pts_host, ext)
    t2 = time.perf_counter()
    keep = oracle.filter_mask(pts_host, pts_host[ring], threads=threads) if len(ring) >= 3 else None
    t3 = time.perf_counter()
    surv = np.flatnonzero(keep) if keep is not None else np.arange(len(pts_host))
    oracle.hull(pts_host, surv)
    t4 = time.perf_counter()
    return {"extremes": round(t1 - t0, 4), "polygon": round(t2 - t1, 6), "filter": round(t3 - t2, 4),
            "hull": round(t4 - t3, 4), "survivors": int(len(surv))}


def cpu_baseline(pts_dev, n_local: int, threads: int, angles: str, config: str, target_s: float = 12.0) -> dict:
    """the oracle as it stands on the host cores -- all cores
    (--threads nproc) and one core pinned to CPU 0 (taskset -c 0), on leading
    samples of the same workload sized for ~target_s seconds each; per-phase
    times; the CPU model."""
    n_s, _ = sized_sample(pts_dev, target_s, threads, angles, min(n_local, 200_000_000))
    host = pts_dev[:n_s].cpu().numpy()
    rate, dt = oracle_rate(host, threads, angles)
    phases = oracle_phases(host, threads, angles)
    # single thread, pinned to CPU 0
    old = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    try:
        if old is not None:
            os.sched_setaffinity(0, {min(old)})
        n1 = max(100_000, min(n_s, int(rate / max(threads, 1) * target_s / 2)))
        h1 = host[:n1]
        rate1, dt1 = oracle_rate(h1, 1, angles)
        phases1 = oracle_phases(h1, 1, angles)
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    return {"value": rate / 1e9, "unit": "Gpts/s", "cores": threads, "kind": "oracle",
            "sample": f"first {n_s} points of {config} (oracle Steps 1-3, {dt:.1f} s, {threads} threads)",
            "per_phase_s": phases, "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
            "single_thread": {"value": rate1 / 1e9, "unit": "Gpts/s", "cores": 1, "pinned": f"cpu {min(old) if old else 0}",
                              "sample": f"first {n1} points ({dt1:.1f} s)", "per_phase_s": phases1}}


def sized_sample(pts_dev, target_s: float, threads: int, angles: str, cap: int):
    """Pick a sample size that takes about target_s seconds of oracle work."""
    pilot = min(cap, 2_000_000)
    rate, _ = oracle_rate(pts_dev[:pilot].cpu().numpy(), threads, angles)
    n = int(min(cap, max(pilot, rate * target_s)))
    return n, rate


METRIC3 = "3D extension (P:115): filtered points/sec (Gpts/s) and % of HBM roofline; discard %"
K13_BYTES_PER_PT = 12         # K1-3D reads each float3 once
K23_BYTES_PER_PT = 12         # K2-3D reads each float3 once ...
K23_BYTES_PER_SURVIVOR = 20   # ... and writes int64 index + float3 point per survivor


def oracle3_rate(pts_host: np.ndarray, threads: int, angles: str):
    import oracle

    oracle.build()
    t0 = time.perf_counter()
    oracle.cudapre3(pts_host, angles, threads=threads)
    dt = time.perf_counter() - t0
    return len(pts_host) / dt, dt


def sized_sample3(pts_dev, target_s: float, threads: int, angles: str, cap: int):
    pilot = min(cap, 200_000)
    rate, _ = oracle3_rate(pts_dev[:pilot].cpu().numpy(), threads, angles)
    return int(min(cap, max(pilot, rate * target_s))), rate


def main3(args, world, rank, local):
    """The 3D extension (configs synth.CONFIGS3, not BASELINE
    configs): one step = K1-3D (+ D2H of the picks; N > 1: all-gather + host
    merge), host Step 2 (polyhedron + cell lists, H2D), K2-3D writing each
    survivor's int64 index and float3 point (+ D2H of the count)."""
    import torch
    import torch.distributed as dist

    import paper_1405_3454_b200 as cp
    import synth
    import synth.cuda as scuda
    from paper_1405_3454_b200 import build as pbuild

    cfg = dict(synth.CONFIGS3[args.config])
    n_total = args.n or cfg.pop("n")
    cfg.pop("n", None)
    family, seed = cfg.pop("family"), cfg.pop("seed")
    threads = os.cpu_count() or 1
    torch.cuda.set_device(local)
    if args.impl == "reference":   # the 3D oracle on a bounded sample, rank 0 only
        if rank != 0:
            return
        scuda.build()
        sample_cap = min(n_total, 20_000_000)
        dev = scuda.generate3(family, sample_cap, seed=seed, **cfg)
        n_s, _ = sized_sample3(dev, 2.0, threads, args.angles, sample_cap)
        host = dev[:n_s].cpu().numpy()
        del dev
        import oracle

        for _ in range(args.warmup):
            oracle.cudapre3(host, args.angles, threads=threads)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle.cudapre3(host, args.angles, threads=threads)
        dt = time.perf_counter() - t0
        v = n_s * args.steps / dt / 1e9
        print(json.dumps({
            "metric": METRIC3, "value": v, "unit": "Gpts/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: {n_total} pts {family} seed {seed}",
                       "sample_points_per_step": n_s},
            "cpu_baseline": {"value": v, "unit": "Gpts/s", "cores": threads, "kind": "oracle",
                             "sample": f"first {n_s} points of {args.config} per step"},
            "e2e": {"value": v, "unit": "Gpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)
        return

    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    if rank == 0:
        pbuild.build()
        scuda.build()
    if group is not None:
        dist.barrier()
    n_local = n_total // world + (1 if rank < n_total % world else 0)
    base = rank * (n_total // world) + min(rank, n_total % world)
    pts = scuda.generate3(family, n_local, seed=seed, base=base, **cfg)
    ws = cp.Workspace3(n_local)
    out_idx = torch.empty(n_local, dtype=torch.int64, device="cuda")
    out_pts = None if args.no_points else torch.empty((n_local, 3), dtype=torch.float32, device="cuda")
    ext_dev = torch.empty(ctypes_sizeof(cp.Extremes3T), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    k1_ms, k2_ms, info = [], [], {}

    def step(timed=True):
        ext = cp.extremes3(pts, args.angles, index_base=base, ws=ws, device_out=ext_dev,
                           timing=k1_ms if timed else None)
        if group is not None:   # cross-rank combine of the Step-1 blocks (as 2D a3)
            ext = cp.exchange3(ext, group, device_buf=ext_dev)
        idx, _, poly = cp.filter3(pts, ext, index_base=base, ws=ws, out_idx=out_idx, out_pts=out_pts,
                                  return_points=out_pts is not None, timing=k2_ms if timed else None)
        info.update(surv=idx.shape[0], nf=poly.nf, exact=ext.raw.exact_points,
                    mean_cand=poly.raw.n_entries / max(1, poly.raw.n_cells), long_cells=poly.raw.long_cells)

    for _ in range(args.warmup):
        step(False)
    clocks = ClockSampler(torch.cuda.current_device())
    if group is not None:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks:
        start.record()
        for _ in range(args.steps):
            step()
        end.record()
        torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    surv = info["surv"]
    if group is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        s_ = torch.tensor([surv], device="cuda", dtype=torch.int64)
        dist.all_reduce(s_)
        surv_total = int(s_.item())
    else:
        surv_total = surv
    value = n_total * args.steps / (ms / 1e3) / 1e9

    pk = peaks()
    peak = pk["hbm_gbs"] if pk else 6650.0
    k1, k2 = statistics.mean(k1_ms), statistics.mean(k2_ms)
    k1_bytes = K13_BYTES_PER_PT * n_local
    k2_bytes = K23_BYTES_PER_PT * n_local + (K23_BYTES_PER_SURVIVOR if out_pts is not None else 8) * surv
    kernels = {"k1_extremes3": (k1, k1_bytes), "k2_filter3": (k2, k2_bytes)}
    dom = max(kernels, key=lambda k: kernels[k][0])
    d_ms, d_bytes = kernels[dom]
    achieved = d_bytes / (d_ms / 1e3) / 1e9
    traffic = None
    try:
        ent = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config, {}).get(dom)
        if ent and int(ent.get("n_local", -1)) == n_local:
            traffic = ent["dram_bytes_per_launch"]
    except (OSError, ValueError):
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, measured)" if pk else "fallback",
                "per_kernel_ms": {k: round(v[0], 4) for k, v in kernels.items()},
                "per_kernel_GBps": {k: round(v[1] / (v[0] / 1e3) / 1e9, 1) for k, v in kernels.items()},
                "pipeline_GBps": round((k1_bytes + k2_bytes) * args.steps / (ms / 1e3) / 1e9, 1)}

    e2e = None
    if not args.no_e2e and group is None:
        e_steps = max(1, min(args.steps, 3))
        try:
            h_pts = torch.empty((n_local, 3), dtype=torch.float32).pin_memory()
            h_surv = torch.empty(n_local, dtype=torch.int64).pin_memory()
        except RuntimeError:
            h_pts = torch.empty((n_local, 3), dtype=torch.float32)
            h_surv = torch.empty(n_local, dtype=torch.int64)
        h_pts.copy_(pts)

        def e2e_step():
            pts.copy_(h_pts, non_blocking=True)
            ext = cp.extremes3(pts, args.angles, index_base=base, ws=ws)
            idx, _, _ = cp.filter3(pts, ext, index_base=base, ws=ws, out_idx=out_idx, return_points=False)
            h_surv[: idx.shape[0]].copy_(idx)
            return idx.shape[0]

        e2e_step()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(e_steps):
            m = e2e_step()
        t1.record()
        torch.cuda.synchronize()
        e_ms = t0.elapsed_time(t1)
        e2e = {"value": n_total * e_steps / (e_ms / 1e3) / 1e9, "unit": "Gpts/s",
               "h2d_bytes_per_step": 12 * n_local, "d2h_bytes_per_step": 8 * m + ctypes_sizeof(cp.Extremes3T) + 8,
               "steps": e_steps, "pinned": bool(h_pts.is_pinned())}
        del h_pts, h_surv

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        n_s, _ = sized_sample3(pts, 12.0, threads, args.angles, min(n_local, 20_000_000))
        rate, dt = oracle3_rate(pts[:n_s].cpu().numpy(), threads, args.angles)
        cpu = {"value": rate / 1e9, "unit": "Gpts/s", "cores": threads, "kind": "oracle",
               "sample": f"first {n_s} points of {args.config} (3D oracle Steps 1-3, {dt:.1f} s)"}

    if rank == 0:
        print(json.dumps({
            "metric": METRIC3, "value": round(value, 3), "unit": "Gpts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {n_total} pts {family} (seed {seed}), float3 AoS, "
                                   f"contiguous shards of {n_local}", "n_total": n_total, "angles": args.angles,
                       "l2": f"inputs larger than L2 ({12 * n_local / 1e9:.2f} GB vs 126 MB), no flush",
                       "parallelism": f"dp{world} (point shards)", "step2": "host (polyhedron + direction cells)"},
            "discard_pct": round(100 * (1 - surv_total / n_total), 4),
            "remaining_pct": round(100 * surv_total / n_total, 4),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": 2 * args.steps, "clocks": clocks.result(),
            "facets": info["nf"], "mean_cell_candidates": round(info["mean_cand"], 3),
            "k1_exact_path_points_per_step": int(info["exact"]),
            "host_step2_and_transfers_ms": round(ms / args.steps - k1 - k2, 4),
        }), flush=True)
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


def ctypes_sizeof(t):
    import ctypes

    return ctypes.sizeof(t)


def main():
    args = parse()
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    import synth

    if args.config in synth.CONFIGS3:
        return main3(args, world, rank, local)

    cfg = dict(synth.CONFIGS[args.config])
    n_total = args.n or cfg.pop("n")
    cfg.pop("n", None)
    family, seed = cfg.pop("family"), cfg.pop("seed")
    threads = os.cpu_count() or 1

    # ------------------------------------------------------------ reference arm: the oracle
    if args.impl == "reference":
        if rank != 0:
            return
        import synth.cuda as scuda

        torch.cuda.set_device(local)
        scuda.build()
        sample_cap = min(n_total, 200_000_000)
        dev = scuda.generate(family, sample_cap, seed=seed, **cfg)
        n_s, _ = sized_sample(dev, 2.0, threads, args.angles, sample_cap)
        host = dev[:n_s].cpu().numpy()
        del dev
        import oracle

        for _ in range(args.warmup):
            oracle.cudapre(host, args.angles, threads=threads)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle.cudapre(host, args.angles, threads=threads)
        dt = time.perf_counter() - t0
        v = n_s * args.steps / dt / 1e9
        line = {"metric": METRIC, "value": v, "unit": "Gpts/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "impl": "reference",
                "config": {"workload": f"{args.config}: {n_total} pts {family} seed {seed}",
                           "sample_points_per_step": n_s},
                "cpu_baseline": {"value": v, "unit": "Gpts/s", "cores": threads, "kind": "oracle",
                                 "sample": f"first {n_s} points of {args.config} per step"},
                "e2e": {"value": v, "unit": "Gpts/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    # ------------------------------------------------------------ our arm
    import torch.distributed as dist

    import paper_1405_3454_b200 as cp
    import synth.cuda as scuda
    from paper_1405_3454_b200 import build as pbuild

    torch.cuda.set_device(local)
    group = comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    if rank == 0:   # (no-op when the in-tree libraries are up to date)
        pbuild.build()
        scuda.build()
    if group is not None:
        dist.barrier()   # no rank loads a library rank 0 may be rebuilding
        comm = cp.Comm.from_group(group)   # the library's own NCCL communicator
    n_local = n_total // world + (1 if rank < n_total % world else 0)
    base = rank * (n_total // world) + min(rank, n_total % world)
    pts = scuda.generate(family, n_local, seed=seed, base=base, **cfg)
    if args.align8:   # the same points at an 8-byte aligned address
        buf = torch.empty((n_local + 1, 2), dtype=torch.float32, device="cuda")
        buf[1:] = pts
        pts = buf[1:]
        assert pts.data_ptr() % 16 == 8
    ws = cp.Workspace(n_local)
    cap = n_local if n_local <= 250_000_000 else n_local // 8   # dense configs (C4) keep ~all points
    out_idx = torch.empty(cap, dtype=torch.int64, device="cuda")
    out_pts = None if args.no_points else torch.empty((cap, 2), dtype=torch.float32, device="cuda")
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    parts = torch.empty(world * cp.EXTREMES_BYTES, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if group is None:
            return v
        t = torch.tensor([v], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # (A) Steps 1-3 on the device (Step 2 by the device builder, SURVEY §8 f3;
    # N > 1: the library's NCCL all-gather of the ranks' Step-1 blocks, merged
    # by the builder): the host only enqueues; CUDA events between the calls
    # time seed+K1, (all-gather +) Step 2 and K2 on their stream.
    def dstep(ev):
        if ev:
            ev[0].record()
        cp.extremes_device(pts, args.angles, index_base=base, ws=ws)
        if ev:
            ev[1].record()
        if comm is not None:
            cp.allgather_extremes(comm, ws, parts)
            cp.polygon_device(ws, parts=parts, nparts=world)
        else:
            cp.polygon_device(ws)
        if ev:
            ev[2].record()
        cp.filter_geom(pts, index_base=base, ws=ws, out_idx=out_idx, out_pts=out_pts, count=count)
        if ev:
            ev[3].record()

    # (B) the paper's host Step 2 between the kernels: N = 1 one library
    # call per step (K1 writes the picks to mapped host memory, the host builds
    # the polygon, one H2D of the geometry, K2; one host wait); N > 1 the
    # all-gather + host merge (cudapre_extremes_comm), then cudapre_filter.
    hpoly = []

    def hstep():
        if comm is None:
            hpoly.clear()
            cp.pipeline_host(pts, args.angles, index_base=base, ws=ws, out_idx=out_idx, out_pts=out_pts,
                             polygon_out=hpoly)
        else:
            ext = cp.extremes_comm(pts, comm, args.angles, index_base=base, ws=ws)
            cp.filter(pts, ext, index_base=base, ws=ws, out_idx=out_idx, out_pts=out_pts,
                      return_points=out_pts is not None)

    def timed(fn, steps, evs=None):
        if group is not None:
            dist.barrier()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for i in range(steps):
            fn(evs[i]) if evs is not None else fn()
        t1.record()
        torch.cuda.synchronize()
        return max_over_ranks(t0.elapsed_time(t1))

    for _ in range(args.warmup):
        dstep(None)
        hstep()
    clocks = ClockSampler(torch.cuda.current_device())
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    with clocks:
        ms = timed(dstep, args.steps, evs)
        surv = int(count.item())
        host_ms = timed(hstep, args.steps)
    k1_ms = [e[0].elapsed_time(e[1]) for e in evs]
    poly_ms = [e[1].elapsed_time(e[2]) for e in evs]
    k2_ms = [e[2].elapsed_time(e[3]) for e in evs]
    launches = args.steps * ((2 if n_local >= 65536 else 1) + 2)   # seed + K1 + Step-2 builder + K2
    # per-step diagnostics (not timed): one reported host-path step
    rep1 = cp.ReportT()
    ext = cp.extremes(pts, args.angles, index_base=base, group=group, ws=ws, report=rep1)
    _, _, rep2 = cp.filter(pts, ext, index_base=base, ws=ws, out_idx=out_idx, out_pts=out_pts,
                           return_points=out_pts is not None)
    assert rep2["survivors"] == surv, (rep2["survivors"], surv)
    exact_pts = ext.raw.exact_points
    surv_total = surv
    if group is not None:
        st = torch.tensor([surv], device="cuda", dtype=torch.int64)
        dist.all_reduce(st)
        surv_total = int(st.item())
    value = n_total * args.steps / (ms / 1e3) / 1e9

    # ------------------------------------------------------------ roofline of the dominant kernel
    pk = peaks()
    peak = pk["hbm_gbs"] if pk else 6650.0
    k1 = statistics.mean(k1_ms)
    k2 = statistics.mean(k2_ms)
    k1_bytes = K1_BYTES_PER_PT * n_local
    k2_bytes = K2_BYTES_PER_PT * n_local + (K2_BYTES_PER_SURVIVOR if out_pts is not None else 8) * surv
    kernels = {"k1_extremes(+seed)": (k1, k1_bytes), "k2_filter": (k2, k2_bytes)}
    dom = max(kernels, key=lambda k: kernels[k][0])
    d_ms, d_bytes = kernels[dom]
    achieved = d_bytes / (d_ms / 1e3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        ent = prof.get(args.config, {}).get(dom)
        if ent and int(ent.get("n_local", -1)) == n_local:
            traffic = ent["dram_bytes_per_launch"]
    except (OSError, ValueError):
        pass
    pipe_bytes = (k1_bytes + k2_bytes) * world
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, measured)" if pk else "fallback",
                "per_kernel_ms": {k: round(v[0], 4) for k, v in kernels.items()},
                "per_kernel_GBps": {k: round(v[1] / (v[0] / 1e3) / 1e9, 1) for k, v in kernels.items()},
                "pipeline_GBps": round(pipe_bytes * args.steps / (ms / 1e3) / 1e9 / world, 1),
                "pipeline_frac_of_8TBps": round(pipe_bytes * args.steps / (ms / 1e3) / 1e12 / world / 8.0, 4)}
    host_step2 = {
        "value": round(n_total * args.steps / (host_ms / 1e3) / 1e9, 3), "unit": "Gpts/s",
        "ms_per_step": round(host_ms / args.steps, 4),
        "pipeline_frac_of_8TBps": round(pipe_bytes * args.steps / (host_ms / 1e3) / 1e12 / world / 8.0, 4),
        "host_polygon_ms": round(hpoly[0][1], 4) if hpoly else round(rep2["ms_polygon_host"], 4),
        "path": ("cudapre_pipeline_host: K1 -> picks in mapped host memory -> host chain + geometry -> "
                 "one H2D -> K2 (one host wait per step)" if comm is None else
                 "cudapre_extremes_comm (NCCL all-gather + host merge) -> cudapre_filter"),
    }

    # ------------------------------------------------------------ N > 1: collecting the survivors
    multi = None
    if comm is not None:
        g_steps = max(1, min(args.steps, 5))
        root_idx = torch.empty(max(1, int(surv_total * 1.01) + 1024) if rank == 0 else 1, dtype=torch.int64,
                               device="cuda")
        root_pts = torch.empty((root_idx.shape[0], 2), dtype=torch.float32, device="cuda") if rank == 0 else None

        def gather_step():
            _, _, c = cp.pipeline_comm(pts, comm, args.angles, index_base=base, ws=ws, out_idx=out_idx,
                                       out_pts=out_pts, parts=parts)
            cp.gather_survivors(comm, out_idx, out_pts, int(c.item()), root=0, out_idx=root_idx, out_pts=root_pts)

        poly_raw = cp.PolygonT()

        def hull_step():
            _, _, c = cp.pipeline_comm(pts, comm, args.angles, index_base=base, ws=ws, out_idx=out_idx,
                                       out_pts=out_pts, parts=parts)
            m = int(c.item())
            ctypes_memmove(poly_raw, ws.tensor[cp.WS_POLY_OFFSET:cp.WS_POLY_OFFSET + ctypes_sizeof(cp.PolygonT)])
            return cp.hull_comm(comm, out_pts, out_idx, m, poly_raw, root=0)

        gather_step()
        ring = hull_step()
        g_ms = timed(gather_step, g_steps)
        h_ms = timed(hull_step, g_steps)
        multi = {"filter_value": round(value, 3),
                 "filter_gather_value": round(n_total * g_steps / (g_ms / 1e3) / 1e9, 3),
                 "filter_gather_ms_per_step": round(g_ms / g_steps, 4),
                 "gathered_bytes_per_step": 16 * surv_total,
                 "filter_hull_value": round(n_total * g_steps / (h_ms / 1e3) / 1e9, 3),
                 "filter_hull_ms_per_step": round(h_ms / g_steps, 4), "hull_vertices": int(len(ring)) if rank == 0 else None,
                 "comm": "in-library NCCL (cudapre_comm_*): Step-1 all-gather; counts all-gather + grouped "
                         "send/recv of the survivors to rank 0; per-rank GPU hulls + vertex gather"}
        del root_idx, root_pts

    # ------------------------------------------------------------ the paper's end to end: hull with / without CudaPre
    hull_e2e = None
    if comm is None and n_local <= 50_000_000 and not args.no_e2e:
        t0 = time.perf_counter()
        ring_all = cp.hull(pts.cpu().numpy())   # without CudaPre: D2H of every point + the host chain
        t_without = time.perf_counter() - t0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        idx_h, sp_h, rep_h = cp.filter(pts, cp.extremes(pts, args.angles, ws=ws), ws=ws, out_idx=out_idx,
                                       out_pts=out_pts if out_pts is not None else torch.empty((cap, 2), device="cuda"))
        ring_dev = cp.hull_device(sp_h, idx_h, idx_h.shape[0], rep_h["polygon"])   # with CudaPre, GPU final hull
        t_with = time.perf_counter() - t0
        t0 = time.perf_counter()
        idx_h, sp_h, rep_h = cp.filter(pts, cp.extremes(pts, args.angles, ws=ws), ws=ws, out_idx=out_idx,
                                       out_pts=out_pts if out_pts is not None else torch.empty((cap, 2), device="cuda"))
        m_h = idx_h.shape[0]
        sidx = idx_h.cpu().numpy()
        ring_host = sidx[cp.hull(sp_h.cpu().numpy())] if m_h else sidx
        t_with_host = time.perf_counter() - t0
        assert ring_dev.tolist() == ring_all.tolist() == ring_host.tolist(), "hull with / without CudaPre"
        hull_e2e = {"without_cudapre_ms": round(1e3 * t_without, 3),
                    "with_cudapre_gpu_hull_ms": round(1e3 * t_with, 3),
                    "with_cudapre_host_hull_ms": round(1e3 * t_with_host, 3),
                    "speedup_gpu_hull": round(t_without / t_with, 2),
                    "speedup_host_hull": round(t_without / t_with_host, 2),
                    "hull_vertices": int(len(ring_all)), "survivors": int(m_h),
                    "note": ("wall clock: without = D2H of every point + cudapre_hull (host monotone chain); "
                             "with = Steps 1-3 + the survivors' hull (cudapre_hull_device, or D2H + cudapre_hull); "
                             "paper Tables 1-2 report 4-6x (GT640 + Qhull): context only")}

    # ------------------------------------------------------------ e2e: host buffers through the API
    e2e = None
    if not args.no_e2e:
        e_steps = max(1, min(args.steps, 3))
        try:
            h_pts = torch.empty((n_local, 2), dtype=torch.float32).pin_memory()
        except RuntimeError:
            h_pts = torch.empty((n_local, 2), dtype=torch.float32)
        h_pts.copy_(pts)
        h_surv = torch.empty(cap, dtype=torch.int64).pin_memory()
        d2h = 0
        if group is None:
            m, _ = cp.run_host(h_pts, pts, out_idx, h_surv, args.angles, ws=ws)   # warm-up
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(e_steps):
                m, _ = cp.run_host(h_pts, pts, out_idx, h_surv, args.angles, ws=ws)
            t1.record()
            torch.cuda.synchronize()
            e_ms = t0.elapsed_time(t1)
            d2h = 8 * m + cp.EXTREMES_BYTES + 8
        else:
            def e2e_step():
                pts.copy_(h_pts, non_blocking=True)
                ext = cp.extremes_comm(pts, comm, args.angles, index_base=base, ws=ws)
                idx, _, _ = cp.filter(pts, ext, index_base=base, ws=ws, out_idx=out_idx,
                                      return_points=False)
                h_surv[: idx.shape[0]].copy_(idx)
                return idx.shape[0]
            e2e_step()
            e_ms = timed(e2e_step, e_steps)
            m = surv
            d2h = 8 * m + world * cp.EXTREMES_BYTES + 8
        e2e = {"value": n_total * e_steps / (e_ms / 1e3) / 1e9, "unit": "Gpts/s",
               "h2d_bytes_per_step": 8 * n_local, "d2h_bytes_per_step": d2h, "steps": e_steps,
               "pinned": bool(h_pts.is_pinned())}
        del h_pts

    # ------------------------------------------------------------ CPU baseline (oracle), rank 0, N=1
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(pts, n_local, threads, args.angles, args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Gpts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {n_total} pts {family} (seed {seed}), "
                                   f"contiguous shards of {n_local}", "n_total": n_total,
                       "angles": args.angles,
                       "l2": (f"inputs larger than L2 ({8 * n_local / 1e9:.2f} GB vs 126 MB), no flush"
                              if 8 * n_local > 126e6 else
                              f"inputs ({8 * n_local / 1e6:.0f} MB) fit in L2: warm-L2 numbers, not a roofline claim"),
                       "parallelism": f"dp{world} (point shards; {cp.EXTREMES_BYTES} B NCCL all-gather per step)",
                       "step2": "device (byte-identical to the host build, SURVEY f3); host_step2: the paper's host Step 2"},
            "discard_pct": round(100 * (1 - surv_total / n_total), 4),
            "remaining_pct": round(100 * surv_total / n_total, 4),
            "roofline": roofline, "host_step2": host_step2, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks.result(),
            "k1_exact_path_points_per_step": int(exact_pts),
            "step2_device_ms": round(statistics.median(poly_ms), 4),
            "k2_lookback_rounds_per_step": int(rep2["lookback_rounds"]),
            "k2_lookback_spins_per_step": int(rep2["lookback_spins"]),
        }
        if multi is not None:
            line["multi_gpu"] = multi
        if hull_e2e is not None:
            line["hull_e2e"] = hull_e2e
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


def ctypes_memmove(dst_struct, src_u8_tensor):
    import ctypes

    buf = src_u8_tensor.cpu().numpy().tobytes()
    ctypes.memmove(ctypes.addressof(dst_struct), buf, len(buf))


if __name__ == "__main__":
    main()
