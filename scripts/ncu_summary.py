"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py gpurun_out/prof_c5.ncu-rep gpurun_out/launches.csv \
        --round r01 --config C5 --n-local 2000000000

Writes profiles/<round>_<config>_ncu.md (key metrics + stall reasons + the
launch list's per-kernel time shares) and merges the per-launch DRAM bytes of
each kernel into profiles/traffic.json (read by bench.py for `traffic`).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of ncu peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp instr"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]
KEY = {"k1_extremes": "k1_extremes(+seed)", "k2_filter": "k2_filter"}


def ncu_csv(rep: str, page: str, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("launches", nargs="?")
    ap.add_argument("--round", required=True, help="round tag of the output files, e.g. r02c (never overwrite another round's summary)")
    ap.add_argument("--config", required=True)
    ap.add_argument("--n-local", type=int, default=2_000_000_000)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    rows = ncu_csv(a.rep, "raw")
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu summary — {a.config}, round {a.round}", "",
             f"source: `{os.path.basename(a.rep)}` (`ncu --set full --clock-control none`, one launch per kernel)",
             "", a.note, ""]
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        name = d["Kernel Name"]
        lines += [f"## `{name[:90]}`", "", "| metric | value |", "|---|---|"]
        for m, label in METRICS:
            if m in hdr:
                lines.append(f"| {label} (`{m}`) | {d[m]} {units[hdr.index(m)]} |")
        st = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(v), k.replace("smsp__average_warps_issue_stalled_", "")
                               .replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        if st:
            lines += ["", "top stall reasons (warps stalled per issued instruction, "
                      "`smsp__average_warps_issue_stalled_*_per_issue_active.ratio`):", ""]
            lines += [f"- {k}: {v:.2f}" for v, k in sorted(st, reverse=True)[:6]]
        lines.append("")
        for short, key in KEY.items():
            if short + "3" in name:   # the 3D kernels (k1_extremes3, k2_filter3): their own keys
                key = short + "3"
            if short in name:
                rb = to_bytes(d["dram__bytes_read.sum"], units[hdr.index("dram__bytes_read.sum")])
                wb = to_bytes(d["dram__bytes_write.sum"], units[hdr.index("dram__bytes_write.sum")])
                traffic.setdefault(a.config, {})[key] = {
                    "dram_bytes_per_launch": rb + wb, "read": rb, "write": wb,
                    "n_local": a.n_local, "round": a.round, "source": os.path.basename(a.rep)}
    if a.launches and os.path.exists(a.launches):
        lines += ["## launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised)", ""]
        tot = collections.Counter()
        cnt = collections.Counter()
        with open(a.launches) as f:
            body = [l for l in f if l.startswith('"')]
        for r in csv.DictReader(io.StringIO("".join(body))):
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = r["Kernel Name"].split("(")[0].split("::")[-1][:60]
            v = float(r["Metric Value"].replace(",", ""))
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                     "msecond": 1e3}.get(r.get("Metric Unit", "us"), 1.0)
            tot[k] += v * scale
            cnt[k] += 1
        s = sum(tot.values()) or 1.0
        lines += ["| kernel | launches | total µs | share |", "|---|---|---|---|"]
        for k, v in tot.most_common():
            lines.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / s:.1f} % |")
        lines.append("")
    out = os.path.join(ROOT, "profiles", f"{a.round}_{a.config}_ncu.md")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
