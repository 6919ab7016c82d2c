"""Quick CUDA-event timing of the 3D path (K1-3D, host Step 2, K2-3D) on a
device-generated workload: python scripts/time3.py [family] [n] [reps] [angles]."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1405_3454_b200 as cp  # noqa: E402
import synth.cuda  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "ball"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1_000_000_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
angles = sys.argv[4] if len(sys.argv) > 4 else "A"
pts = synth.cuda.generate3(fam, n, seed=23)
ws = cp.Workspace3(n)
out_idx = torch.empty(n, dtype=torch.int64, device="cuda")
out_pts = torch.empty((n, 3), dtype=torch.float32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for r in range(reps + 2):
    torch.cuda.synchronize()
    ev[0].record()
    ext = cp.extremes3(pts, angles, ws=ws)
    ev[1].record()
    idx, _, poly = cp.filter3(pts, ext, ws=ws, out_idx=out_idx, out_pts=out_pts)
    ev[2].record()
    torch.cuda.synchronize()
    t1, t2 = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    m = idx.shape[0]
    print(f"{fam} n={n:.3g} K1+D2H {t1:.3f} ms ({12*n/t1/1e6:.0f} GB/s)  Step2+K2+D2H {t2:.3f} ms "
          f"({(12*n + 20*m)/t2/1e6:.0f} GB/s)  survivors {m} ({100*m/n:.2f}%)  facets {poly.nf} "
          f"entries {poly.raw.n_entries} exact_K1 {ext.raw.exact_points}  total {n/(t1+t2)/1e6:.1f} Gpts/s",
          flush=True)
