"""ctypes binding of librd.so (include/rd.h): argument marshalling only.

Every step of the detection path runs in the CUDA kernels of csrc/; this module only
converts Python/PyTorch objects into the plain pointers and sizes of the C ABI.  There
is no CPU fallback: if librd.so is missing or fails to load, import raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RD_LIB_PATH") or os.path.join(_HERE, "librd.so")   # override: tuning builds

RD_OK, RD_ERR_PARAM, RD_ERR_DIM, RD_ERR_CONFIG, RD_ERR_CAPACITY, RD_ERR_CUDA, RD_ERR_STATE = range(7)
RD_U8, RD_U16 = 0, 1


class rd_config(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("pixel", C.c_int32), ("max_value", C.c_int32),
                ("smoothing_sigma", C.c_double), ("curvature_threshold", C.c_double),
                ("r_min", C.c_int32), ("r_max", C.c_int32), ("vote_threshold_raw", C.c_int32),
                ("vote_threshold_norm", C.c_double), ("sig_a", C.c_int32), ("sig_b", C.c_int32),
                ("sig_den", C.c_int32), ("annulus_halfwidth", C.c_int32), ("max_rings_per_frame", C.c_int32),
                ("max_ridges_per_tile", C.c_int32), ("max_entries_per_tile", C.c_int32),
                ("max_hotspots_per_level", C.c_int32), ("debug", C.c_int32), ("feature", C.c_int32),
                ("edge_threshold", C.c_double)]


RING_DTYPE = np.dtype([("cx", "i4"), ("cy", "i4"), ("r", "i4"), ("raw_votes", "i4"), ("score_fixed", "i8"),
                       ("inliers", "i4"), ("fit_ok", "i4"), ("fx", "f8"), ("fy", "f8"), ("fr", "f8"),
                       ("rms", "f8")])
RIDGE_DTYPE = np.dtype([("x", "i4"), ("y", "i4"), ("dx", "f8"), ("dy", "f8")])
HOT_DTYPE = np.dtype([("r", "i4"), ("y", "i4"), ("x", "i4"), ("raw", "i4"), ("S", "i8")])
STATS_DTYPE = np.dtype([("ridges", "i8"), ("votes", "i8"), ("hotspots", "i8"), ("peaks", "i8")])
FPR_DTYPE = np.dtype([("r", "i4"), ("pad", "i4"), ("votes", "i8"), ("sq", "i8"), ("pos", "i8")])
assert RING_DTYPE.itemsize == 64 and FPR_DTYPE.itemsize == 32
RD_HOST_DEPTH = 2   # host-path calls in flight (rd_submit_host)
RD_DUMP_RIDGES, RD_DUMP_LEVEL_FPR, RD_DUMP_HOTSPOTS, RD_DUMP_MEMBERS = range(4)
OVF_BITS = {"ridges": 1, "entries": 2, "hotspots": 4, "rings": 8, "debug": 16, "output": 32}


class rd_overflow(C.Structure):
    _fields_ = [("frames_overflowed", C.c_int32), ("flags", C.c_int32), ("needed_ridges_per_tile", C.c_int32),
                ("needed_entries_per_tile", C.c_int32), ("needed_hotspots_per_level", C.c_int32),
                ("needed_rings_per_frame", C.c_int32), ("needed_rings_total", C.c_int64)]

EXPORTS = ("rd_abi_version", "rd_status_string", "rd_last_error", "rd_config_init", "rd_create", "rd_destroy",
           "rd_detect", "rd_detect_host", "rd_submit_host", "rd_wait_host", "rd_sync", "rd_query_overflow", "rd_query_flags", "rd_get_stats",
           "rd_debug_dump", "rd_eigen", "rd_set_timing", "rd_kernel_times", "rd_phase_cycles", "rd_ring_members")


class RDError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = lib().rd_status_string(status).decode()
        if status == RD_ERR_CUDA:
            msg += ": " + lib().rd_last_error().decode()
        super().__init__(f"{where}: {msg} (status {status})")


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.rd_abi_version.restype = i32
        L.rd_status_string.argtypes = [C.c_int]
        L.rd_status_string.restype = C.c_char_p
        L.rd_last_error.restype = C.c_char_p
        L.rd_config_init.argtypes = [C.POINTER(rd_config), i32, i32, i32]
        L.rd_create.argtypes = [C.POINTER(rd_config), i32, i32, C.POINTER(vp)]
        L.rd_destroy.argtypes = [vp]
        L.rd_detect.argtypes = [vp, vp, i64, i64, i32, vp, i32, vp, vp, vp]
        L.rd_detect_host.argtypes = [vp, vp, i64, i64, i32, vp, i32, vp, vp]
        L.rd_submit_host.argtypes = [vp, vp, i64, i64, i32, vp, i32, vp, vp]
        L.rd_wait_host.argtypes = [vp]
        L.rd_sync.argtypes = [vp]
        L.rd_query_overflow.argtypes = [vp, C.POINTER(rd_overflow)]
        L.rd_query_flags.argtypes = [vp, i32, vp]
        L.rd_get_stats.argtypes = [vp, i32, vp]
        L.rd_debug_dump.argtypes = [vp, i32, i32, vp, i64, C.POINTER(i64)]
        L.rd_eigen.argtypes = [vp, i64, vp, vp, vp]
        L.rd_set_timing.argtypes = [vp, i32]
        L.rd_kernel_times.argtypes = [vp, vp, C.POINTER(i32)]
        L.rd_phase_cycles.argtypes = [vp, i32, vp]
        L.rd_ring_members.argtypes = [vp, i32, vp, i32, vp, i64, C.POINTER(i64)]
        for n in EXPORTS:
            if n not in ("rd_abi_version", "rd_status_string", "rd_last_error"):
                getattr(L, n).restype = C.c_int
        _LIB = L
    return _LIB


def check(status, where):
    if status != RD_OK:
        raise RDError(status, where)


def make_config(width, height, pixel_bytes, **kw) -> rd_config:
    c = rd_config()
    check(lib().rd_config_init(C.byref(c), width, height, RD_U8 if pixel_bytes == 1 else RD_U16), "rd_config_init")
    for name, _ in rd_config._fields_:
        if name in kw and kw[name] is not None:
            setattr(c, name, kw[name])
    return c
