"""Speculative pre-filter check on the BASELINE configs:
survivors with the pre-filter (first Step 3 after Step 1) == survivors of a
plain streaming Step 3 (a second Step 3: the candidates are consumed) ==
the oracle (configs the oracle finishes quickly), plus CUDA-event timings of
both.  python scripts/spec_check.py [C2a C2b C3 C4 C4e0 C5]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1405_3454_b200 as cp  # noqa: E402
import synth  # noqa: E402
import synth.cuda as scuda  # noqa: E402

names = sys.argv[1:] or ["C2a", "C2b", "C3", "C4", "C4e0", "C5"]
scuda.build()
for name in names:
    cfg = dict(synth.CONFIGS[name])
    n = cfg.pop("n")
    fam, seed = cfg.pop("family"), cfg.pop("seed")
    pts = scuda.generate(fam, n, seed=seed, **cfg)
    ws = cp.Workspace(n)
    cap = n if n <= 250_000_000 else n // 8
    oi = torch.empty(cap, dtype=torch.int64, device="cuda")
    op = torch.empty((cap, 2), dtype=torch.float32, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    res = {}
    for rep in range(4):
        torch.cuda.synchronize()
        ev[0].record()
        ext = cp.extremes(pts, "A", ws=ws)
        ev[1].record()
        idx, sp, r = cp.filter(pts, ext, ws=ws, out_idx=oi, out_pts=op)
        ev[2].record()
        info = cp.spec_info(ws)
        if rep == 0:
            a = (idx.cpu().numpy(), sp.cpu().numpy())
        torch.cuda.synchronize()
        ev[3].record()
        idx2, sp2, r2 = cp.filter(pts, ext, ws=ws, out_idx=oi, out_pts=op)   # no candidates left: streaming
        torch.cuda.synchronize()
        ev[0].synchronize()
        info2 = cp.spec_info(ws)
        t_k1 = ev[0].elapsed_time(ev[1])
        t_k2 = ev[1].elapsed_time(ev[2])
        if rep == 0:
            b = (idx2.cpu().numpy(), sp2.cpu().numpy())
            same = np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            res["same"] = same
        res.setdefault("k1", []).append(t_k1)
        res.setdefault("k2spec", []).append(t_k2)
        res.setdefault("k2raw", []).append(r2["ms_filter_kernel"])
    print(f"{name}: n={n} surv={len(a[0])} ({100*len(a[0])/n:.3f}%) spec={info} raw_used={info2['used']} "
          f"same={res['same']} K1 {np.median(res['k1']):.4f} ms  Step2+3(spec) {np.median(res['k2spec']):.4f} ms  "
          f"K2 raw kernels {np.median(res['k2raw']):.4f} ms  cand_frac={info['candidates']/n:.4f}", flush=True)
    if n <= 50_000_000 and os.environ.get("ORACLE", "1") == "1":
        import oracle
        t0 = time.time()
        want = oracle.cudapre(pts.cpu().numpy(), "A", threads=os.cpu_count())
        ok = np.array_equal(a[0], want["survivors"])
        print(f"  oracle: {ok} ({time.time()-t0:.1f} s)", flush=True)
        assert ok
    assert res["same"]
    del pts, ws, oi, op
    torch.cuda.empty_cache()
