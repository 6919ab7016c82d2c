"""Device twin of ``synth.generate``: writes the same bytes straight into HBM."""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "gen.cu")
LIB = os.path.join(_HERE, "libsynth.so")
_FAM = {"square": 0, "disk": 1, "gauss": 2, "circle": 3, "cube": 10, "ball": 11, "sphere": 12}
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-O3", "-fmad=false", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
                               "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} missing: run synth.cuda.build()")
        L = ctypes.CDLL(LIB)
        L.synth_generate.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_ulonglong,
                                     ctypes.c_longlong, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]
        L.synth_generate.restype = ctypes.c_int
        _lib = L
    return _lib


def generate_into(out, family: str, seed: int, base: int = 0, *, lo: float = -1.0, hi: float = 1.0,
                  eps: float = 1e-3, stream=None):
    """Fill the CUDA float32 tensor ``out`` ((n, 2), or (n, 3) for a 3D family)
    with points [base, base+n)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    rc = _load().synth_generate(_FAM[family], out.shape[0], seed, base, lo, hi, eps,
                                ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_generate failed with CUDA error {rc}")
    return out


def generate(family: str, n: int, seed: int, base: int = 0, device="cuda", **kw):
    import torch

    out = torch.empty((n, 2), dtype=torch.float32, device=device)
    return generate_into(out, family, seed, base, **kw)


def generate3(family: str, n: int, seed: int, base: int = 0, device="cuda", **kw):
    import torch

    out = torch.empty((n, 3), dtype=torch.float32, device=device)
    return generate_into(out, family, seed, base, **kw)
