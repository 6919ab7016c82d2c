"""Phase timing of the device polygon builder (perf experiment only): build
with -DCUDAPRE_GEOM_TIMING=1, which writes clock64 deltas just below the
geometry page (inside the workspace header page)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1405_3454_b200 as cp
import synth
xy = synth.generate("disk", 10_000_000, seed=3)
pts = torch.from_numpy(xy).cuda()
ws = cp.Workspace(len(xy))
for _ in range(5):
    cp.extremes_device(pts, "A", ws=ws)
    cp.polygon_device(ws)
torch.cuda.synchronize()
t = ws.tensor[cp.WS_GEOM_OFFSET - 512: cp.WS_GEOM_OFFSET].cpu().view(torch.int64).tolist()
names = ["phase A + defaults", "edges + box search", "disk", "sector prep", "sample rays", "buckets", "finish"]
for i, n in enumerate(names):
    print(f"{n:22s} {t[i + 1] / 1965:.1f} us")
print(f"  of which: stage ext {t[8] / 1965:.1f} us, chain {t[9] / 1965:.1f} us, defaults {t[10] / 1965:.1f} us")
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(100):
    cp.polygon_device(ws)
e.record(); torch.cuda.synchronize()
print(f"polygon_device launch: {s.elapsed_time(e) / 100 * 1000:.1f} us per call")
