"""Run under torchrun (one process per GPU): the multi-GPU paths of the public
API against the oracle on the whole set.

1. torch.distributed group path: cp.cuda_pre(..., group) (NCCL all-gather of
   the per-rank Step-1 structs + host merge), survivors concatenated in rank
   order;
2. the device-resident path: K1 -> NCCL all-gather of the workspace Step-1
   blocks -> merge + Step 2 on the device -> K2;
3. the in-library NCCL communicator (cudapre_comm_*): cudapre_extremes_comm
   (host merge), cudapre_pipeline_comm (Steps 1-3 on the stream), the survivor
   gather to rank 0 (cudapre_gather_survivors) and the sharded final hull
   (cudapre_hull_comm);
4. the 3D extension over NCCL.
Prints "nccl ok" on rank 0 when every check passed."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
import paper_1405_3454_b200 as cp  # noqa: E402
import synth  # noqa: E402

N = int(os.environ.get("NCCL_TEST_N", "3000017"))


def shard(n, rank, world):
    n_local = n // world + (1 if rank < n % world else 0)
    base = rank * (n // world) + min(rank, n % world)
    return n_local, base


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    n_local, base = shard(N, rank, world)
    xy = synth.generate("disk", n_local, seed=6, base=base)
    pts = torch.from_numpy(xy).cuda()
    # 1. torch.distributed group path
    idx, sp, rep = cp.cuda_pre(pts, "A", group=dist.group.WORLD, index_base=base)
    counts = [None] * world
    dist.all_gather_object(counts, idx.cpu().numpy())
    # 2. device-resident path over torch's NCCL
    ws = cp.Workspace(n_local)
    gathered = torch.empty(world * cp.EXTREMES_BYTES, dtype=torch.uint8, device="cuda")
    cp.extremes_device(pts, "A", index_base=base, ws=ws)
    dist.all_gather_into_tensor(gathered, cp.result_view(ws), group=dist.group.WORLD)
    cp.polygon_device(ws, parts=gathered, nparts=world)
    d_idx = torch.empty(n_local, dtype=torch.int64, device="cuda")
    d_count = torch.zeros(1, dtype=torch.int64, device="cuda")
    cp.filter_geom(pts, index_base=base, ws=ws, out_idx=d_idx, count=d_count)
    torch.cuda.synchronize()
    assert np.array_equal(d_idx[: int(d_count.item())].cpu().numpy(), idx.cpu().numpy()), "device path"
    # 3. the in-library communicator
    comm = cp.Comm.from_group(dist.group.WORLD)
    assert (comm.rank, comm.world) == (rank, world)
    ext_c = cp.extremes_comm(pts, comm, "A", index_base=base)
    assert ext_c.idx.tolist() == rep["extremes"].idx.tolist(), "extremes_comm"
    o_idx, o_pts, o_cnt = cp.pipeline_comm(pts, comm, "A", index_base=base)
    torch.cuda.synchronize()
    m = int(o_cnt.item())
    assert np.array_equal(o_idx[:m].cpu().numpy(), idx.cpu().numpy()), "pipeline_comm"
    assert np.array_equal(o_pts[:m].cpu().numpy(), xy[o_idx[:m].cpu().numpy() - base]), "pipeline_comm points"
    g_idx, g_pts, g_tot = cp.gather_survivors(comm, o_idx, o_pts, m, root=0)
    # collective errors: every rank returns the same status, none waits in a
    # send / receive — a NULL d_idx on the last rank, then a root that takes
    # points while the last rank passes none
    L = cp.lib()
    total = cp.ctypes.c_int64()
    last = rank == world - 1
    r_idx = torch.empty(max(g_tot, 1), dtype=torch.int64, device="cuda") if rank == 0 else None
    r_pts = torch.empty((max(g_tot, 1), 2), dtype=torch.float32, device="cuda") if rank == 0 else None
    vp = cp.ctypes.c_void_p
    for bad_idx, bad_pts in ((True, False), (False, True)):
        st = L.cudapre_gather_survivors(
            comm.handle, None if (last and bad_idx) else vp(o_idx.data_ptr()),
            None if (last and bad_pts) else vp(o_pts.data_ptr()), max(m, 1), 0,
            vp(r_idx.data_ptr()) if rank == 0 else None, vp(r_pts.data_ptr()) if rank == 0 else None,
            max(g_tot, 1), None, cp.ctypes.byref(total))
        assert st == cp.ERR_ARG, (rank, bad_idx, bad_pts, st)
    # capacity: every rank sees CAPACITY and the total it needs
    st = L.cudapre_gather_survivors(comm.handle, vp(o_idx.data_ptr()), None, m, 0,
                                    vp(r_idx.data_ptr()) if rank == 0 else None, None, 0, None,
                                    cp.ctypes.byref(total))
    assert (st == cp.ERR_CAPACITY) == (g_tot > 0) and total.value == g_tot, (rank, st, total.value)
    poly = cp.polygon(ext_c)
    ring_c = cp.hull_comm(comm, o_pts, o_idx, m, poly, root=0)
    # an empty shard on the last rank (world > 1): extremes_comm still gives the global answer
    if world > 1:
        e_local, e_base = (n_local, base) if rank < world - 1 else (0, N)
        e_pts = pts if rank < world - 1 else torch.empty((0, 2), dtype=torch.float32, device="cuda")
        ext_e = cp.extremes_comm(e_pts, comm, "A", index_base=e_base)
        assert ext_e.n == N - shard(N, world - 1, world)[0], "empty-shard extremes_comm"
    # pipeline_comm with an empty shard on the last rank (world 1: the only one)
    e_pts = pts if rank < world - 1 else torch.empty((0, 2), dtype=torch.float32, device="cuda")
    e_base = base if rank < world - 1 else N
    pe_idx, _, pe_cnt = cp.pipeline_comm(e_pts, comm, "A", index_base=e_base, return_points=False)
    torch.cuda.synchronize()
    pe = pe_idx[: int(pe_cnt.item())].cpu().numpy()
    if rank == world - 1:
        assert len(pe) == 0, "empty shard: no survivors"
    pe_all = [None] * world
    dist.all_gather_object(pe_all, pe)
    # 4. the 3D extension
    n3 = N // 3
    n3_local, base3 = shard(n3, rank, world)
    xyz = synth.generate3("ball", n3_local, seed=7, base=base3)
    p3 = torch.from_numpy(xyz).cuda()
    dev3 = torch.empty(cp.ctypes.sizeof(cp.Extremes3T), dtype=torch.uint8, device="cuda")
    local3 = cp.extremes3(p3, "A", index_base=base3, device_out=dev3)
    ext3 = cp.exchange3(local3, dist.group.WORLD, device_buf=dev3)
    idx3, _, poly3 = cp.filter3(p3, ext3, index_base=base3, return_points=False)
    parts3 = [None] * world
    dist.all_gather_object(parts3, idx3.cpu().numpy())
    if rank == 0:
        got = np.concatenate(counts)
        full = synth.generate("disk", N, seed=6)
        want = oracle.cudapre(full, "A", threads=os.cpu_count())
        assert rep["extremes"].idx.tolist() == want["ext_idx"].tolist(), "Step 1"
        assert np.array_equal(got, want["survivors"]), "Step 3"
        assert g_tot == len(want["survivors"]), "gather total"
        assert np.array_equal(g_idx.cpu().numpy(), want["survivors"]), "gathered survivors"
        assert np.array_equal(g_pts.cpu().numpy(), full[want["survivors"]]), "gathered points"
        assert ring_c.tolist() == oracle.hull(full).tolist(), "hull_comm"
        n_e = N - shard(N, world - 1, world)[0]   # the set without the last shard
        if n_e > 0:
            want_e = oracle.cudapre(full[:n_e], "A", threads=os.cpu_count())
            assert np.array_equal(np.concatenate(pe_all), want_e["survivors"]), "pipeline_comm, empty last shard"
        full3 = synth.generate3("ball", n3, seed=7)
        want3 = oracle.cudapre3(full3, "A", threads=os.cpu_count())
        assert ext3.idx.tolist() == want3["ext_idx"].tolist(), "3D Step 1"
        assert poly3.facets.tolist() == want3["facets"].tolist(), "3D Step 2"
        assert np.array_equal(np.concatenate(parts3), want3["survivors"]), "3D Step 3"
        print(f"nccl ok world={world} survivors={len(got)} gathered={g_tot} hull={len(ring_c)} "
              f"3d={len(want3['survivors'])}")
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
