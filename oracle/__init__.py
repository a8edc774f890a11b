"""ctypes binding of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py.  The product package paper_1310_1371_b200 never
imports this module, and the oracle shares no code with it.  See oracle.h for the
paper passages each function follows.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class Params(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("pixel_bytes", C.c_int32),
                ("smoothing_sigma", C.c_double), ("curvature_threshold", C.c_double),
                ("r_min", C.c_int32), ("r_max", C.c_int32), ("vote_threshold_raw", C.c_int32),
                ("vote_threshold_norm", C.c_double), ("sig_a", C.c_int32), ("sig_b", C.c_int32),
                ("sig_den", C.c_int32), ("annulus_halfwidth", C.c_int32), ("feature", C.c_int32),
                ("edge_threshold", C.c_double)]


RIDGE_DTYPE = np.dtype([("x", "i4"), ("y", "i4"), ("dx", "f8"), ("dy", "f8"), ("kappa", "f8")])
HOT_DTYPE = np.dtype([("r", "i4"), ("y", "i4"), ("x", "i4"), ("raw", "i4"), ("S", "i8")])
RING_DTYPE = np.dtype([("cx", "i4"), ("cy", "i4"), ("r", "i4"), ("raw_votes", "i4"), ("score_fixed", "i8"),
                       ("inliers", "i4"), ("fit_ok", "i4"), ("fx", "f8"), ("fy", "f8"), ("fr", "f8"),
                       ("rms", "f8")])
STATS_DTYPE = np.dtype([("ridges", "i8"), ("votes", "i8"), ("hotspots", "i8"), ("peaks", "i8")])


def lib():
    global _LIB
    if _LIB is None:
        # ORACLE_LIB_PATH: a mutated build (tools/mutate_oracle.py checks that the pins catch it)
        path = os.environ.get("ORACLE_LIB_PATH") or os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            from tools.build import build_oracle
            build_oracle()
        L = C.CDLL(path)
        P = C.POINTER(Params)
        L.orc_gauss_taps.argtypes = [C.c_double, C.c_void_p, C.c_int32]
        L.orc_gauss_taps.restype = C.c_int32
        for name in ("orc_level_halfwidth", "orc_annulus_halfwidth"):
            getattr(L, name).argtypes = [P, C.c_int32]
            getattr(L, name).restype = C.c_int32
        L.orc_level_weight.argtypes = [P, C.c_int32, C.c_int32]
        L.orc_level_weight.restype = C.c_int32
        L.orc_sigma.argtypes = [P, C.c_int32]
        L.orc_sigma.restype = C.c_double
        L.orc_norm_threshold.argtypes = [P, C.c_int32]
        L.orc_norm_threshold.restype = C.c_double
        L.orc_curvature_threshold_int.argtypes = [P]
        L.orc_curvature_threshold_int.restype = C.c_double
        L.orc_edge_threshold_int2.argtypes = [P]
        L.orc_edge_threshold_int2.restype = C.c_double
        L.orc_gradient.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_gradient.restype = None
        L.orc_smooth.argtypes = [P, C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_hessian.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_eigen.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_double)]
        L.orc_eigen.restype = C.c_int
        L.orc_ridges.argtypes = [P, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
        L.orc_ridges.restype = C.c_int64
        L.orc_votes.argtypes = [P, C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_votes.restype = C.c_int64
        L.orc_window_sum.argtypes = [P, C.c_void_p, C.c_int32, C.c_int32, C.c_int32]
        L.orc_window_sum.restype = C.c_int64
        L.orc_detect.argtypes = [P, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_int64]
        L.orc_detect.restype = C.c_int64
        L.orc_detect_batch.argtypes = [P, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                       C.c_void_p, C.c_int32]
        L.orc_detect_batch.restype = C.c_int
        L.orc_detect_batch_streamed.argtypes = L.orc_detect_batch.argtypes
        L.orc_pool_create.argtypes = [P, C.c_int32, C.c_int32]
        L.orc_pool_create.restype = C.c_void_p
        L.orc_pool_detect.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32,
                                      C.c_void_p, C.c_void_p]
        L.orc_pool_detect.restype = C.c_int
        L.orc_pool_free.argtypes = [C.c_void_p]
        L.orc_detect_batch_streamed.restype = C.c_int
        L.orc_peaks.argtypes = [P, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        L.orc_peaks.restype = C.c_int64
        L.orc_stream_peaks.argtypes = [P, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                       C.POINTER(C.c_int64)]
        L.orc_stream_peaks.restype = C.c_int64
        L.orc_fit.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32] + [C.POINTER(C.c_double)] * 4
        L.orc_fit.restype = C.c_int
        _LIB = L
    return _LIB


def params(**kw) -> Params:
    p = Params()
    for name, _ in Params._fields_:
        if name in kw:
            setattr(p, name, kw[name])
    return p


def _img(p: Params, img: np.ndarray) -> np.ndarray:
    img = np.ascontiguousarray(img)
    assert img.shape == (p.height, p.width)
    assert img.dtype == (np.uint8 if p.pixel_bytes == 1 else np.uint16)
    return img


def gauss_taps(sigma: float) -> np.ndarray:
    t = np.zeros(256, dtype=np.int32)
    K = lib().orc_gauss_taps(sigma, t.ctypes.data, 256)
    return t[: 2 * K + 1].copy()


def level_halfwidth(p, r):
    return lib().orc_level_halfwidth(C.byref(p), r)


def level_weight(p, r, d):
    return lib().orc_level_weight(C.byref(p), r, d)


def sigma(p, r):
    return lib().orc_sigma(C.byref(p), r)


def norm_threshold(p, r):
    return lib().orc_norm_threshold(C.byref(p), r)


def curvature_threshold_int(p):
    return lib().orc_curvature_threshold_int(C.byref(p))


def annulus_halfwidth(p, r):
    return lib().orc_annulus_halfwidth(C.byref(p), r)


def smooth(p, img) -> np.ndarray:
    img = _img(p, img)
    G = np.zeros((p.height, p.width), dtype=np.float64)
    lib().orc_smooth(C.byref(p), img.ctypes.data, img.strides[0], G.ctypes.data)
    return G


def hessian(p, G):
    G = np.ascontiguousarray(G, dtype=np.float64)
    out = [np.zeros((p.height, p.width), dtype=np.float64) for _ in range(3)]
    lib().orc_hessian(C.byref(p), G.ctypes.data, *[o.ctypes.data for o in out])
    return tuple(out)  # Ixx, Iyy, Ixy


def gradient(p, G):
    """Edge variant (NEXT-2, R19): 5x5 first-order Sobel gradient (Ix, Iy) of G."""
    G = np.ascontiguousarray(G, dtype=np.float64)
    Ix, Iy = (np.zeros((p.height, p.width), dtype=np.float64) for _ in range(2))
    lib().orc_gradient(C.byref(p), G.ctypes.data, Ix.ctypes.data, Iy.ctypes.data)
    return Ix, Iy


def edge_threshold_int2(p):
    return lib().orc_edge_threshold_int2(C.byref(p))


def eigen(a, b, c):
    k, dx, dy = C.c_double(), C.c_double(), C.c_double()
    deg = lib().orc_eigen(a, b, c, C.byref(k), C.byref(dx), C.byref(dy))
    return k.value, dx.value, dy.value, bool(deg)


def ridges(p, img) -> np.ndarray:
    img = _img(p, img)
    cap = p.width * p.height
    out = np.zeros(cap, dtype=RIDGE_DTYPE)
    n = lib().orc_ridges(C.byref(p), img.ctypes.data, img.strides[0], out.ctypes.data, cap)
    if n < 0:
        raise RuntimeError("orc_ridges failed")
    return out[:n].copy()


def n_levels(p):
    return p.r_max - p.r_min + 3


def votes(p, ridge_arr) -> tuple[np.ndarray, int]:
    ridge_arr = np.ascontiguousarray(ridge_arr, dtype=RIDGE_DTYPE)
    raw = np.zeros((n_levels(p), p.height, p.width), dtype=np.int32)
    n = lib().orc_votes(C.byref(p), ridge_arr.ctypes.data, len(ridge_arr), raw.ctypes.data)
    return raw, n


def window_sum(p, raw, r, y, x) -> int:
    raw = np.ascontiguousarray(raw, dtype=np.int32)
    assert raw.shape == (n_levels(p), p.height, p.width)
    return lib().orc_window_sum(C.byref(p), raw.ctypes.data, r, y, x)


def peaks(p, raw):
    """Steps 6-8 on a given raw accumulator [N_r, H, W] -> (peaks, hotspots) as HOT_DTYPE arrays."""
    raw = np.ascontiguousarray(raw, dtype=np.int32)
    assert raw.shape == (n_levels(p), p.height, p.width)
    pk = np.zeros(4096, dtype=HOT_DTYPE)
    hcap = max(1024, int((raw > p.vote_threshold_raw).sum()))
    hot = np.zeros(hcap, dtype=HOT_DTYPE)
    nh = C.c_int64()
    n = lib().orc_peaks(C.byref(p), raw.ctypes.data, pk.ctypes.data, len(pk), hot.ctypes.data, hcap, C.byref(nh))
    if n < 0:
        raise RuntimeError("orc_peaks failed")
    return pk[:n].copy(), hot[: nh.value].copy()


def stream_peaks(p, ridge_arr, hot_cap: int = 1 << 21):
    """The paper's streamed steps 5-8 (SI steps 2-4) on a ridge list -> (peaks, hotspots)."""
    ridge_arr = np.ascontiguousarray(ridge_arr, dtype=RIDGE_DTYPE)
    pk = np.zeros(4096, dtype=HOT_DTYPE)
    hot = np.zeros(hot_cap, dtype=HOT_DTYPE)
    nh = C.c_int64()
    n = lib().orc_stream_peaks(C.byref(p), ridge_arr.ctypes.data, len(ridge_arr), pk.ctypes.data, len(pk),
                               hot.ctypes.data, hot_cap, C.byref(nh))
    if n < 0:
        raise RuntimeError("orc_stream_peaks failed")
    return pk[: min(n, len(pk))].copy(), hot[: min(nh.value, hot_cap)].copy()


def detect(p, img, want_debug=False):
    """Returns (rings, stats[, ridges, hotspots])."""
    img = _img(p, img)
    ring_cap = 4096
    rings = np.zeros(ring_cap, dtype=RING_DTYPE)
    st = np.zeros(1, dtype=STATS_DTYPE)
    if want_debug:
        rcap = p.width * p.height
        rid = np.zeros(rcap, dtype=RIDGE_DTYPE)
        hcap = 1 << 21
        hot = np.zeros(hcap, dtype=HOT_DTYPE)
        n = lib().orc_detect(C.byref(p), img.ctypes.data, img.strides[0], rings.ctypes.data, ring_cap,
                             st.ctypes.data, rid.ctypes.data, rcap, hot.ctypes.data, hcap)
    else:
        n = lib().orc_detect(C.byref(p), img.ctypes.data, img.strides[0], rings.ctypes.data, ring_cap,
                             st.ctypes.data, None, 0, None, 0)
    if n < 0:
        raise RuntimeError("orc_detect failed (bad parameters or allocation)")
    s = st[0]
    res = (rings[: min(n, ring_cap)].copy(), s)
    if want_debug:
        res = res + (rid[: s["ridges"]].copy(), hot[: min(s["hotspots"], hcap)].copy())
    return res


def detect_batch(p, frames: np.ndarray, nthreads: int = 0, ring_stride: int = 1024, streamed: bool = False):
    """Steps 1-10 on many frames with a host thread pool.  streamed=True does steps 5-8 the
    paper's streamed way (oracle/streamed.c); the outputs are identical."""
    frames = np.ascontiguousarray(frames)
    n = frames.shape[0]
    rings = np.zeros((n, ring_stride), dtype=RING_DTYPE)
    counts = np.zeros(n, dtype=np.int32)
    stats = np.zeros(n, dtype=STATS_DTYPE)
    fn = lib().orc_detect_batch_streamed if streamed else lib().orc_detect_batch
    rc = fn(C.byref(p), frames.ctypes.data, frames.strides[0], n, rings.ctypes.data,
                                ring_stride, counts.ctypes.data, stats.ctypes.data, nthreads)
    if rc:
        raise RuntimeError("orc_detect_batch failed")
    return [rings[i, : counts[i]].copy() for i in range(n)], stats


class Pool:
    """Host thread pool with per-thread workspaces kept across calls (orc_pool_*): the same
    outputs as detect_batch; only the allocation of the full arrays is paid once."""

    def __init__(self, p, nthreads: int = 0, streamed: bool = False):
        self.p = p
        self._h = lib().orc_pool_create(C.byref(p), nthreads, 1 if streamed else 0)
        if not self._h:
            raise RuntimeError("orc_pool_create failed")

    def detect(self, frames: np.ndarray, ring_stride: int = 1024):
        frames = np.ascontiguousarray(frames)
        n = frames.shape[0]
        rings = np.zeros((n, ring_stride), dtype=RING_DTYPE)
        counts = np.zeros(n, dtype=np.int32)
        stats = np.zeros(n, dtype=STATS_DTYPE)
        if lib().orc_pool_detect(self._h, frames.ctypes.data, frames.strides[0], n, rings.ctypes.data, ring_stride,
                                 counts.ctypes.data, stats.ctypes.data):
            raise RuntimeError("orc_pool_detect failed")
        return [rings[i, : counts[i]].copy() for i in range(n)], stats

    def close(self):
        if self._h:
            lib().orc_pool_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fit(xs, ys, cx, cy):
    xs = np.ascontiguousarray(xs, dtype=np.int32)
    ys = np.ascontiguousarray(ys, dtype=np.int32)
    out = [C.c_double() for _ in range(4)]
    ok = lib().orc_fit(xs.ctypes.data, ys.ctypes.data, len(xs), cx, cy, *[C.byref(o) for o in out])
    return bool(ok), tuple(o.value for o in out)
