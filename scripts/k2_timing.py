"""Per-warp cycle breakdown of the TMA K2 kernel (perf experiment only).

Runs Steps 1-3 on a synthetic config with CUDAPRE_K2_DEBUG=2, which selects
the instrumented kernel build; lane 0 of every warp accumulates clock64()
deltas per phase and the kernel adds them into the workspace header page at
kWsDbgOffset.  Prints the per-warp totals of the last launch in
microseconds-per-block terms.

  CUDAPRE_K2_DEBUG=2 python scripts/k2_timing.py --config C5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

DBG_OFFSET = 2048
PHASES = ["passA", "barrierA", "resolve/scan", "barrierB", "emit"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--points", action="store_true", help="also write survivor coordinates (as bench.py)")
    args = ap.parse_args()
    if os.environ.get("CUDAPRE_K2_DEBUG") != "2":
        print("(CUDAPRE_K2_DEBUG != 2: only the dense-emit counter is meaningful)")
    import torch

    import paper_1405_3454_b200 as cp
    import synth
    import synth.cuda as scuda

    cfg = dict(synth.CONFIGS[args.config])
    family, n, seed = cfg.pop("family"), cfg.pop("n"), cfg.pop("seed")
    pts = scuda.generate(family, n, seed=seed, base=0, **cfg)
    ws = cp.Workspace(n)
    cap = max(1024, n // 8)
    out_idx = torch.empty(cap, dtype=torch.int64, device="cuda")
    out_pts = torch.empty((cap, 2), dtype=torch.float32, device="cuda") if args.points else None
    for _ in range(args.runs):
        ws.tensor[DBG_OFFSET:DBG_OFFSET + 384].zero_()
        ext = cp.extremes(pts, "A", ws=ws)
        idx, _, rep = cp.filter(pts, ext, ws=ws, out_idx=out_idx, out_pts=out_pts, return_points=args.points)
        torch.cuda.synchronize()
    d = ws.tensor[DBG_OFFSET:DBG_OFFSET + 384].cpu().view(torch.int64).tolist()
    clk = torch.cuda.get_device_properties(0).clock_rate * 1e3 if hasattr(
        torch.cuda.get_device_properties(0), "clock_rate") else 1.9e9
    blocks = 2 * torch.cuda.get_device_properties(0).multi_processor_count
    print(f"dense (list-overflow) warp emits in the last launch: {d[44]}")
    print(f"K2 {rep['ms_filter_kernel']:.3f} ms, survivors {idx.shape[0]}, blocks {blocks}, clock {clk/1e9:.2f} GHz")
    us = lambda c: c / clk / blocks * 1e6
    print("per-block average, microseconds (cycles / clock / blocks)")
    print("compute warp    passA   buffer-wait")
    for w in range(8):
        print(f"{w:12d} {us(d[w]):8.1f} {us(d[8 + w]):12.1f}")
    print("emit warp: " + ", ".join(f"{n} {us(d[16 + i]):.1f}" for i, n in
                                    enumerate(["wait tile_done", "scan+publish", "resolve", "emit"])))

if __name__ == "__main__":
    main()
