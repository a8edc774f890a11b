"""Seeded synthetic ring frames (ctypes binding of synth/libsynth.so).

INPUT module shared by the oracle tests, the CUDA parity tests and bench.py.  It
holds none of the detection method's arithmetic — only ring layouts, Gaussian
profile rendering and noise (BASELINE.json configs).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .presets import EDGE_THRESHOLD, PRESETS, edge_preset, preset  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class SynthRing(C.Structure):
    _fields_ = [("cx", C.c_double), ("cy", C.c_double), ("r", C.c_double), ("amp", C.c_double),
                ("occ_start", C.c_double), ("occ_len", C.c_double), ("group", C.c_int32), ("kind", C.c_int32)]


class SynthScene(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("pixel_bytes", C.c_int32),
                ("max_value", C.c_int32), ("background", C.c_double), ("sigma_p", C.c_double),
                ("read_sigma", C.c_double), ("poisson", C.c_int32)]


RING_DTYPE = np.dtype([("cx", "f8"), ("cy", "f8"), ("r", "f8"), ("amp", "f8"), ("occ_start", "f8"),
                       ("occ_len", "f8"), ("group", "i4"), ("kind", "i4")])
assert RING_DTYPE.itemsize == C.sizeof(SynthRing)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            from tools.build import build_synth
            build_synth()
        L = C.CDLL(path)
        L.synth_config_shape.argtypes = [C.c_int] + [C.POINTER(C.c_int32)] * 5
        L.synth_config_scene.argtypes = [C.c_int, C.POINTER(SynthScene)]
        L.synth_layout.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_void_p, C.c_int32]
        L.synth_render.argtypes = [C.POINTER(SynthScene), C.c_void_p, C.c_int32, C.c_uint64, C.c_void_p, C.c_int64]
        L.synth_frame.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32,
                                  C.POINTER(C.c_int32)]
        L.synth_batch.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int32, C.c_void_p, C.c_int32]
        L.synth_u01.argtypes = [C.c_uint64, C.c_uint64]
        L.synth_u01.restype = C.c_double
        L.synth_key.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.synth_key.restype = C.c_uint64
        _LIB = L
    return _LIB


def config_shape(cfg: int):
    v = [C.c_int32() for _ in range(5)]
    if lib().synth_config_shape(cfg, *[C.byref(x) for x in v]):
        raise ValueError(f"unknown config {cfg}")
    W, H, pb, mv, batch = (x.value for x in v)
    return dict(width=W, height=H, pixel_bytes=pb, max_value=mv, batch=batch,
                dtype=np.uint8 if pb == 1 else np.uint16)


def config_scene(cfg: int) -> SynthScene:
    s = SynthScene()
    if lib().synth_config_scene(cfg, C.byref(s)):
        raise ValueError(f"unknown config {cfg}")
    return s


def scene(width, height, pixel_bytes=1, max_value=255, background=20.0, sigma_p=1.0, read_sigma=0.0, poisson=0):
    return SynthScene(width, height, pixel_bytes, max_value, background, sigma_p, read_sigma, poisson)


def layout(cfg: int, seed: int, idx: int) -> np.ndarray:
    out = np.zeros(1024, dtype=RING_DTYPE)
    n = lib().synth_layout(cfg, seed, idx, out.ctypes.data, len(out))
    if n < 0:
        raise ValueError("layout failed")
    return out[:n].copy()


def render(sc: SynthScene, rings, noise_key: int = 0) -> np.ndarray:
    rings = np.ascontiguousarray(rings, dtype=RING_DTYPE)
    dt = np.uint8 if sc.pixel_bytes == 1 else np.uint16
    out = np.zeros((sc.height, sc.width), dtype=dt)
    if lib().synth_render(C.byref(sc), rings.ctypes.data, len(rings), noise_key, out.ctypes.data,
                          sc.width * sc.pixel_bytes):
        raise RuntimeError("render failed")
    return out


def make_rings(spec) -> np.ndarray:
    """spec: iterable of (cx, cy, r, amp[, occ_start, occ_len])."""
    out = np.zeros(len(spec), dtype=RING_DTYPE)
    for i, s in enumerate(spec):
        out[i]["cx"], out[i]["cy"], out[i]["r"], out[i]["amp"] = s[:4]
        if len(s) > 4:
            out[i]["occ_start"], out[i]["occ_len"] = s[4], s[5]
        out[i]["group"] = -1
    return out


def frame(cfg: int, seed: int, idx: int):
    sh = config_shape(cfg)
    img = np.zeros((sh["height"], sh["width"]), dtype=sh["dtype"])
    truth = np.zeros(1024, dtype=RING_DTYPE)
    n = C.c_int32()
    if lib().synth_frame(cfg, seed, idx, img.ctypes.data, truth.ctypes.data, len(truth), C.byref(n)):
        raise RuntimeError("synth_frame failed")
    return img, truth[: n.value].copy()


def batch(cfg: int, seed: int, first: int, n: int, nthreads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    sh = config_shape(cfg)
    if out is None:
        out = np.empty((n, sh["height"], sh["width"]), dtype=sh["dtype"])
    assert out.flags.c_contiguous and out.shape == (n, sh["height"], sh["width"]) and out.dtype == sh["dtype"]
    if lib().synth_batch(cfg, seed, first, n, out.ctypes.data, nthreads):
        raise RuntimeError("synth_batch failed")
    return out


def u01(key: int, counter: int) -> float:
    return lib().synth_u01(key, counter)
