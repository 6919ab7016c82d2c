"""The multi-GPU ABI's host-side behaviour on a CPU-only box (no CUDA device):
NCCL is loaded at run time and makes its 128-byte id; every entry point
rejects bad arguments before touching a device or NCCL; the Python wrapper's
structure sizes match the C header.  The collectives themselves run under
torchrun on GPUs (tests/scripts/nccl_cudapre.py)."""
import ctypes

import pytest

import paper_1405_3454_b200 as cp


def test_unique_id_is_128_distinct_bytes():
    a, b = cp.Comm.unique_id(), cp.Comm.unique_id()
    assert len(a) == len(b) == 128
    assert a != b and any(a)


@pytest.mark.parametrize("rank,world", [(2, 2), (-1, 2), (0, 0)])
def test_create_rejects_bad_ranks(rank, world):
    L = cp.lib()
    h = ctypes.c_void_p()
    st = L.cudapre_comm_create(ctypes.create_string_buffer(cp.Comm.unique_id(), 128), rank, world,
                               ctypes.byref(h))
    assert st == cp.ERR_ARG and not h.value
    assert b"rank" in L.cudapre_last_error()
    with pytest.raises(ValueError):
        cp.Comm(0, 1, b"short")


def test_entry_points_reject_a_null_comm():
    L = cp.lib()
    total = ctypes.c_int64()
    assert L.cudapre_gather_survivors(None, None, None, 0, 0, None, None, 0, None, ctypes.byref(total)) == cp.ERR_ARG
    assert L.cudapre_comm_allgather_extremes(None, None, None, None) == cp.ERR_ARG
    ring_len = ctypes.c_int64()
    poly = cp.PolygonT()
    assert L.cudapre_hull_comm(None, None, None, 0, ctypes.byref(poly), None, 0, 0, None, None, 0,
                               ctypes.byref(ring_len)) == cp.ERR_ARG
    r, w = ctypes.c_int32(), ctypes.c_int32()
    assert L.cudapre_comm_rank(None, ctypes.byref(r), ctypes.byref(w)) == cp.ERR_ARG
    assert L.cudapre_comm_destroy(None) == cp.OK


def test_status_codes_match_the_header():
    import os
    import re

    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                            "cudapre.h")).read()
    codes = dict((m[0], int(m[1])) for m in re.findall(r"(CUDAPRE_ERR_\w+|CUDAPRE_OK) = (\d+)", hdr))
    assert codes["CUDAPRE_ERR_NCCL"] == cp.ERR_NCCL == 7
    assert codes["CUDAPRE_ERR_CAPACITY"] == cp.ERR_CAPACITY
