"""Multi-rank path on CPU (world_size 2, gloo): the cross-rank exchange and
merge of Step-1 results gives every rank the single-set
answer and the same polygon.  On GPUs the same ``cp.exchange`` runs over NCCL
straight from the device buffer K1 writes; the host logic is identical.

Per-rank Step-1 structs come from the ORACLE here (no GPU on this box)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

N = 40_001


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cuts, out_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import paper_1405_3454_b200 as cp
    import synth
    from tests.test_abi import _ext_from_oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        lo, hi = cuts[rank], cuts[rank + 1]
        xy = synth.generate("disk", hi - lo, seed=6, base=lo)      # this rank's shard only
        local = _ext_from_oracle(oracle, xy, base=lo)
        merged = cp.exchange(local, dist.group.WORLD)
        poly = cp.polygon(merged)
        out_q.put((rank, merged.idx.tolist(), poly.vidx.tolist(), merged.n))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cuts", [[0, 17_000, N], [0, N, N], [0, 1, N]])
def test_two_rank_exchange_matches_single(cuts, oracle_lib):
    import synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cuts, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    xy = synth.generate("disk", N, seed=6)
    want = oracle_lib.cudapre(xy, "A")
    for rank, idx, ring, n in res:
        assert n == N
        assert idx == want["ext_idx"].tolist(), rank
        assert ring == want["ring"].tolist(), rank


def _worker3(rank, world, port, cuts, out_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1405_3454_b200 as cp
    import synth
    from tests.test_abi3 import _ext3_from_oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        lo, hi = cuts[rank], cuts[rank + 1]
        xyz = np.round(synth.generate3("ball", hi - lo, seed=6, base=lo) * 32).astype(np.float32)   # ties
        local = _ext3_from_oracle(xyz, "A")
        for j in range(24):
            if local.raw.idx[j] >= 0:
                local.raw.idx[j] += lo
        merged = cp.exchange3(local, dist.group.WORLD)
        poly = cp.polyhedron3(merged)
        out_q.put((rank, merged.idx.tolist(), poly.facets.tolist(), merged.n))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cuts", [[0, 17_000, N], [0, 1, N]])
def test_two_rank_exchange3_matches_single(cuts, oracle_lib):
    """3D: the all-gathered, merged Step-1 structs equal the oracle's
    single-set picks on every rank, and so do the facets built from them."""
    import synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker3, args=(r, 2, port, cuts, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    xyz = np.round(synth.generate3("ball", N, seed=6) * 32).astype(np.float32)
    want = oracle_lib.cudapre3(xyz, "A")
    for rank, idx, facets, n in res:
        assert n == N
        assert idx == want["ext_idx"].tolist(), rank
        assert facets == want["facets"].tolist(), rank
