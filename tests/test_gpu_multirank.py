"""Multi-rank path with the product's own Step-1 structs (K1 on the GPU), two
processes sharing cuda:0 and exchanging over gloo (host memory): every rank
merges the other rank's K1 result with the library's lexicographic rule,
builds the same polygon and filters its shard; the concatenated survivors,
the picks and the polygon equal the oracle's on the whole set.

The ranks' kernels never wait on each other (the exchange is a host
all-gather between independent launches), so this is not a stand-in for
NCCL over several GPUs; the NCCL transport is tests/scripts/nccl_cudapre.py
(torchrun, one process per GPU)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, family, cuts, out_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import paper_1405_3454_b200 as cp
    import synth

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        lo, hi = cuts[rank], cuts[rank + 1]
        xy = synth.generate(family, hi - lo, seed=12, base=lo)
        pts = torch.from_numpy(xy).cuda() if hi > lo else torch.empty((0, 2), dtype=torch.float32, device="cuda")
        idx, sp, rep = cp.cuda_pre(pts, "A", group=dist.group.WORLD, index_base=lo)
        parts = [None] * world
        dist.all_gather_object(parts, (idx.cpu().numpy(), sp.cpu().numpy() if sp is not None else None))
        if rank == 0:
            out_q.put((rep["extremes"].idx.tolist(), rep["polygon"].vidx.tolist(),
                       np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("family,n,cut", [("disk", 2_000_003, 0.37), ("square", 1_000_001, 0.5),
                                          ("circle", 500_009, 0.9), ("disk", 300_007, 1.0)])
def test_two_ranks_product_structs(family, n, cut):
    import oracle
    import synth

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1405_3454_b200 import build

    build.build()
    cuts = [0, int(n * cut), n]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, family, cuts, q)) for r in range(2)]
    for p in procs:
        p.start()
    ext_idx, ring, surv, surv_pts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    xy = synth.generate(family, n, seed=12)
    want = oracle.cudapre(xy, "A", threads=os.cpu_count())
    assert ext_idx == want["ext_idx"].tolist()
    assert ring == want["ring"].tolist()
    assert np.array_equal(surv, want["survivors"])
    assert np.array_equal(surv_pts, xy[want["survivors"]])
