"""Build libcudapre.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1405_3454_b200.build [--force] [--verbose]

Host C++ is compiled with -ffp-contract=off (exact predicates);
device code never relies on contraction either way (explicit __*_rn intrinsics).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcudapre.so")
BUILD = os.path.join(HERE, "_build")
SOURCES = ["api.cpp", "host_geom.cpp", "k1_extremes.cu", "k2_filter.cu", "k2_filter_tma.cu",
           "k_polygon.cu", "k_hull.cu",
           # the 3D extension
           "api3.cpp", "host_geom3.cpp", "comm.cpp", "k1_extremes3.cu", "k2_filter3.cu"]
# per-file extra flags: the device polygon builder must not contract multiply-adds (it has to agree
# bit for bit with the host builder, compiled with -ffp-contract=off)
EXTRA = {"k_polygon.cu": ["-fmad=false"]}
HEADERS = ["internal.h", "device.h", "exact.cuh", "geom.cuh", "k2_common.cuh", "tma.cuh", "internal3.h", "exact3.cuh",
           os.path.join("..", "..", "include", "cudapre.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
              "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s, *hdrs]):
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, *EXTRA.get(src, []), "-c", s, "-o", o]
            if verbose and src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
            if verbose or res.returncode:
                sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            if res.returncode:
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode:
            raise RuntimeError("link failed:\n" + res.stdout + res.stderr)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
