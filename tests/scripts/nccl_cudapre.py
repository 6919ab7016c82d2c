"""Run under torchrun: each rank filters its contiguous shard through the
public API with group=WORLD (NCCL all-gather of the per-rank Step-1 structs),
then rank 0 gathers the survivors and checks them against the oracle."""
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


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    n_local = N // world + (1 if rank < N % world else 0)
    base = rank * (N // world) + min(rank, N % world)
    xy = synth.generate("disk", n_local, seed=6, base=base)
    pts = torch.from_numpy(xy).cuda()
    idx, sp, rep = cp.cuda_pre(pts, "A", group=dist.group.WORLD, index_base=base)
    counts = [None] * world
    dist.all_gather_object(counts, idx.cpu().numpy())
    # device-resident path: K1 -> NCCL all-gather of the workspace's Step-1
    # blocks -> merge + Step 2 on the device -> K2, no host round trip
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
    # the 3D extension: K1-3D writes its Step-1 block to a device
    # buffer, NCCL all-gathers the blocks, the host merges them (cp.exchange3)
    n3 = N // 3
    n3_local = n3 // world + (1 if rank < n3 % world else 0)
    base3 = rank * (n3 // world) + min(rank, n3 % world)
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
        full3 = synth.generate3("ball", n3, seed=7)
        want3 = oracle.cudapre3(full3, "A", threads=os.cpu_count())
        assert ext3.idx.tolist() == want3["ext_idx"].tolist(), "3D Step 1"
        assert poly3.facets.tolist() == want3["facets"].tolist(), "3D Step 2"
        assert np.array_equal(np.concatenate(parts3), want3["survivors"]), "3D Step 3"
        print(f"nccl ok world={world} survivors={len(got)} 3d={len(want3['survivors'])}")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
