"""bench.py keeps the driver's JSON contract (one line; metric, value, unit,
n_gpus, steps, warmup, ms_per_step, higher_is_better, scaling, vs_baseline,
dtype, data, config; roofline, cpu_baseline, e2e, gpu_launches, clocks) for
the 2D path, the 3D extension and the reference arm — on small configs so the
test takes seconds."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("args", [("--config", "C2b"), ("--config", "T1")])
def test_bench_line_contract(args):
    d = _run(*args, "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert BASE_KEYS <= d.keys()
    assert d["value"] > 0 and d["unit"] == "Gpts/s" and d["n_gpus"] == 1
    assert d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["scaling"] in ("weak", "strong") and d["data"] == "synthetic"
    assert "workload" in d["config"]
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys()
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= e.keys()
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert "cpu_baseline" in d and 0 <= d["discard_pct"] <= 100
    if args[1] == "C2b":   # the paper's host Step 2 and end-to-end hull with / without CudaPre
        h = d["host_step2"]
        assert h["value"] > 0 and h["ms_per_step"] > 0 and 0 < h["pipeline_frac_of_8TBps"]
        he = d["hull_e2e"]
        assert he["without_cudapre_ms"] > 0 and he["with_cudapre_gpu_hull_ms"] > 0 and he["hull_vertices"] >= 3


def test_bench_cpu_baseline_fields():
    """cpu_baseline: all cores and one pinned core, per-phase
    times, the CPU model."""
    d = _run("--config", "C1", "--steps", "3", "--warmup", "3", "--no-e2e")
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["value"] > 0 and c["cores"] >= 1 and c["cpu_model"]
    assert c["single_thread"]["cores"] == 1 and c["single_thread"]["value"] > 0
    assert {"extremes", "polygon", "filter", "hull"} <= c["per_phase_s"].keys()


def test_bench_reference_arm_contract():
    d = _run("--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "1")
    assert BASE_KEYS <= d.keys() and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "Gpts/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
