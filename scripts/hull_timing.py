"""Time the GPU final hull (f1) against the host chain on the survivors."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1405_3454_b200 as cp
import synth.cuda as scuda

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
pts = scuda.generate("disk", n, seed=6)
idx, sp, rep = cp.cuda_pre(pts, "A")
m = idx.shape[0]
cp.hull_device(sp, idx, m, rep["polygon"])            # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
ring, rem = cp.hull_device(sp, idx, m, rep["polygon"], return_remaining=True)
t1 = time.perf_counter()
h_pts = sp.cpu().numpy()
h_ids = idx.cpu().numpy()
t2 = time.perf_counter()
ring2 = cp.hull(h_pts, np.arange(m))                  # host chain on every survivor
t3 = time.perf_counter()
assert ring.tolist() == h_ids[ring2].tolist()
print(f"n={n} survivors={m} left for the host chain={rem} hull={len(ring)} vertices")
print(f"GPU final hull {1e3 * (t1 - t0):.1f} ms; host chain on all survivors {1e3 * (t3 - t2):.1f} ms")
