"""Detector: Python face of rd_create / rd_detect / rd_detect_host / rd_submit_host (include/rd.h).

Argument marshalling only: every step of the path runs in librd.so's CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _rd
from ._rd import FPR_DTYPE, HOT_DTYPE, RIDGE_DTYPE, RING_DTYPE, STATS_DTYPE, check, lib

_CFG_KEYS = ("max_value", "smoothing_sigma", "curvature_threshold", "r_min", "r_max", "vote_threshold_raw",
             "vote_threshold_norm", "sig_a", "sig_b", "sig_den", "annulus_halfwidth", "max_rings_per_frame",
             "max_ridges_per_tile", "max_entries_per_tile", "max_hotspots_per_level", "debug", "feature",
             "edge_threshold")


@dataclass
class RingBatch:
    """Output of one detect call (rd.h: rings of frame f are rings[offsets[f]:offsets[f] + counts[f]],
    canonical (r, cy, cx) order; counts[f] = -1 if a capacity overflowed for frame f).
    rings: [capacity, 64] uint8 records (device tensor or host array/tensor)."""
    rings: object
    counts: object
    offsets: object

    def __iter__(self):   # (rings, counts, offsets) unpacking
        return iter((self.rings, self.counts, self.offsets))

    def to_numpy(self) -> list:
        """Per-frame structured arrays (RING_DTYPE); None for frames with count -1."""
        def host(x):
            return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
        c, o = host(self.counts), host(self.offsets)
        r = host(self.rings)
        r = r.reshape(-1).view(np.uint8).view(RING_DTYPE) if r.dtype != RING_DTYPE else r.reshape(-1)
        return [r[o[i]:o[i] + c[i]].copy() if c[i] >= 0 else None for i in range(len(c))]


class Detector:
    """One rd_detector on one CUDA device.

    params: width, height, pixel_bytes plus any rd_config field (see include/rd.h).
    """

    def __init__(self, params: dict, max_batch: int = 1, device: int = 0):
        self.params = dict(params)
        self.width, self.height = int(params["width"]), int(params["height"])
        self.pixel_bytes = int(params["pixel_bytes"])
        self.max_batch = int(max_batch)
        self.device = int(device)
        self.cfg = _rd.make_config(self.width, self.height, self.pixel_bytes,
                                   **{k: params[k] for k in _CFG_KEYS if k in params})
        self.ring_cap = self.cfg.max_rings_per_frame or 1024
        h = C.c_void_p()
        check(lib().rd_create(C.byref(self.cfg), self.max_batch, self.device, C.byref(h)), "rd_create")
        self._h = h

    @classmethod
    def sized_for(cls, params: dict, frames: torch.Tensor, max_batch: int | None = None, device: int = 0,
                  margin: float = 1.25, rounds: int = 4) -> "Detector":
        """A detector whose capacities fit `frames` (a representative CUDA batch): detect, read the
        capacities the call needed (rd_query_overflow) and recreate with them plus a margin until
        nothing overflows.  Capacities change the shared-memory layout and hence the Hough tiling,
        and the needs depend on the tiling, so this iterates (at most `rounds` times)."""
        keys = {"needed_ridges_per_tile": "max_ridges_per_tile", "needed_entries_per_tile": "max_entries_per_tile",
                "needed_hotspots_per_level": "max_hotspots_per_level", "needed_rings_per_frame": "max_rings_per_frame"}
        p = dict(params)
        n = frames.shape[0] if frames.dim() == 3 else 1
        for _ in range(rounds):
            det = cls(p, max_batch=max_batch or n, device=device)
            det.detect(frames)
            det.sync(raise_on_overflow=False)
            ov = det.overflow()
            if ov["frames_overflowed"] == 0:
                return det
            for need, cfg_key in keys.items():
                cur = getattr(det.cfg, cfg_key)
                if cfg_key == "max_hotspots_per_level" and cur == 0:   # automatic (rd_create)
                    cur = 256 if det.cfg.feature == 1 else 160
                if ov[need] > cur:
                    p[cfg_key] = int(ov[need] * margin) + 1
            det.close()
        raise RuntimeError(f"capacities still overflow after {rounds} rounds: {ov}")

    def close(self):
        if getattr(self, "_h", None):
            lib().rd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def frame_dtype(self):
        return torch.uint8 if self.pixel_bytes == 1 else torch.uint16

    def default_capacity(self, n: int) -> int:
        """Output capacity used when the caller gives none: every frame's peak capacity."""
        return n * self.ring_cap

    def alloc_outputs(self, n: int, capacity: int | None = None) -> RingBatch:
        dev = torch.device("cuda", self.device)
        cap = self.default_capacity(n) if capacity is None else int(capacity)
        return RingBatch(torch.empty((max(cap, 1), RING_DTYPE.itemsize), dtype=torch.uint8, device=dev),
                         torch.empty((n,), dtype=torch.int32, device=dev),
                         torch.empty((n + 1,), dtype=torch.int32, device=dev))

    def detect(self, frames: torch.Tensor, out: RingBatch | None = None,
               stream: torch.cuda.Stream | None = None) -> RingBatch:
        """frames: CUDA tensor [N, H, W] (uint8/uint16, row-contiguous).  Asynchronous on `stream`
        (default: torch's current stream).  Returns the RingBatch written (out, or a new one)."""
        if frames.dim() == 2:
            frames = frames.unsqueeze(0)
        n, H, W = frames.shape
        assert (H, W) == (self.height, self.width) and frames.dtype == self.frame_dtype and frames.is_cuda
        assert frames.stride(2) == 1
        if out is None:
            out = self.alloc_outputs(n)
        assert out.counts.numel() >= n and out.offsets.numel() >= n + 1
        st = stream if stream is not None else torch.cuda.current_stream(frames.device)
        es = frames.element_size()
        check(lib().rd_detect(self._h, frames.data_ptr(), frames.stride(1) * es, frames.stride(0) * es, n,
                              out.rings.data_ptr(), out.rings.shape[0], out.counts.data_ptr(), out.offsets.data_ptr(),
                              C.c_void_p(st.cuda_stream)), "rd_detect")
        return out

    def _host_args(self, frames, out, capacity):
        if isinstance(frames, torch.Tensor):
            assert not frames.is_cuda
            ptr, n = frames.data_ptr(), frames.shape[0]
            es = frames.element_size()
            pitch, fstride = frames.stride(1) * es, frames.stride(0) * es
        else:
            if frames.ndim != 3 or frames.strides[2] != frames.itemsize:
                frames = np.ascontiguousarray(frames)
            ptr, n = frames.ctypes.data, frames.shape[0]
            pitch, fstride = frames.strides[1], frames.strides[0]
        if out is None:
            cap = self.default_capacity(n) if capacity is None else int(capacity)
            out = RingBatch(np.empty(max(cap, 1), dtype=RING_DTYPE), np.empty(n, dtype=np.int32),
                            np.empty(n + 1, dtype=np.int32))

        def ptr_of(x):
            return x.data_ptr() if isinstance(x, torch.Tensor) else x.ctypes.data
        args = (self._h, ptr, pitch, fstride, n, ptr_of(out.rings), out.rings.shape[0], ptr_of(out.counts),
                ptr_of(out.offsets))
        return frames, out, args

    def detect_host(self, frames, out: RingBatch | None = None, capacity: int | None = None) -> RingBatch:
        """End-to-end on host buffers (numpy or CPU torch tensor, pinned recommended): the library
        copies frames in, detects and returns the compacted rings, overlapping copies with compute.
        Returns RingBatch of host arrays (rings as RING_DTYPE records)."""
        frames, out, args = self._host_args(frames, out, capacity)
        st = lib().rd_detect_host(*args)
        if st not in (_rd.RD_OK, _rd.RD_ERR_CAPACITY):
            check(st, "rd_detect_host")
        return out

    def submit_host(self, frames, out: RingBatch | None = None, capacity: int | None = None) -> RingBatch:
        """Pipelined detect_host (rd_submit_host): enqueues the call and returns at once; the
        returned RingBatch is filled by the wait_host() that completes this call (calls complete in
        submission order, at most _rd.RD_HOST_DEPTH in flight).  `frames` is kept referenced
        until then."""
        frames, out, args = self._host_args(frames, out, capacity)
        check(lib().rd_submit_host(*args), "rd_submit_host")
        if not hasattr(self, "_pending"):
            self._pending = []
        self._pending.append((frames, out))
        return out

    def wait_host(self) -> RingBatch:
        """Completes the oldest submit_host call (rd_wait_host) and returns its RingBatch."""
        st = lib().rd_wait_host(self._h)
        frames, out = self._pending.pop(0) if getattr(self, "_pending", None) else (None, None)
        if st not in (_rd.RD_OK, _rd.RD_ERR_CAPACITY):
            check(st, "rd_wait_host")
        return out

    def sync(self, raise_on_overflow=True):
        st = lib().rd_sync(self._h)
        if st == _rd.RD_ERR_CAPACITY and not raise_on_overflow:
            return st
        check(st, "rd_sync")
        return st

    def overflow(self) -> dict:
        """rd_query_overflow of the last call: overflowed frames, OR of their bits, needed capacities."""
        o = _rd.rd_overflow()
        check(lib().rd_query_overflow(self._h, C.byref(o)), "rd_query_overflow")
        return {name: getattr(o, name) for name, _ in _rd.rd_overflow._fields_}

    def flags(self, n: int) -> np.ndarray:
        out = np.zeros(n, np.int32)
        check(lib().rd_query_flags(self._h, n, out.ctypes.data), "rd_query_flags")
        return out

    def stats(self, n: int) -> np.ndarray:
        out = np.zeros(n, STATS_DTYPE)
        check(lib().rd_get_stats(self._h, n, out.ctypes.data), "rd_get_stats")
        return out

    def _dump(self, frame: int, what: int, dtype) -> np.ndarray:
        n = C.c_int64()
        check(lib().rd_debug_dump(self._h, frame, what, None, 0, C.byref(n)), "rd_debug_dump")
        out = np.zeros(n.value, dtype)
        check(lib().rd_debug_dump(self._h, frame, what, out.ctypes.data if n.value else None, out.nbytes,
                                  C.byref(n)), "rd_debug_dump")
        return out

    def dump_ridges(self, frame: int) -> np.ndarray:
        return self._dump(frame, _rd.RD_DUMP_RIDGES, RIDGE_DTYPE)

    def dump_hotspots(self, frame: int) -> np.ndarray:
        return self._dump(frame, _rd.RD_DUMP_HOTSPOTS, HOT_DTYPE)

    def dump_level_fpr(self, frame: int) -> np.ndarray:
        return self._dump(frame, _rd.RD_DUMP_LEVEL_FPR, FPR_DTYPE)

    def ring_members(self, frame: int) -> list[np.ndarray]:
        """Classification of frame `frame` of the last detect(): per ring (output order), the
        ridge pixels in its annulus as an (m, 2) int32 array of (x, y), in ridge-bin order."""
        n = C.c_int64()
        cnt = int(self.stats(frame + 1)["peaks"][frame])
        off = np.zeros(cnt + 1, np.int32)
        check(lib().rd_ring_members(self._h, frame, off.ctypes.data, cnt + 1, None, 0, C.byref(n)), "rd_ring_members")
        mem = np.zeros(max(n.value, 1), np.uint32)
        check(lib().rd_ring_members(self._h, frame, off.ctypes.data, cnt + 1, mem.ctypes.data, n.value, C.byref(n)),
              "rd_ring_members")
        xy = np.stack([mem[: n.value] & 0xFFFF, mem[: n.value] >> 16], axis=1).astype(np.int32)
        return [xy[off[i]:off[i + 1]] for i in range(cnt)]

    def set_timing(self, on: bool):
        check(lib().rd_set_timing(self._h, 1 if on else 0), "rd_set_timing")

    def kernel_times(self):
        """(ms per kernel [K1 ridges, K1.5 rays, K2 hough, K3 fit + output] summed over timed calls, n_calls)."""
        ms = (C.c_float * 4)()
        n = C.c_int32()
        check(lib().rd_kernel_times(self._h, ms, C.byref(n)), "rd_kernel_times")
        return [ms[0], ms[1], ms[2], ms[3]], n.value


def eigen(abc: torch.Tensor):
    """Step A3 on device: abc [n, 3] float64 CUDA (Ixx, Ixy, Iyy) -> (kappa_dxdy [n,3], degenerate [n])."""
    assert abc.is_cuda and abc.dtype == torch.float64 and abc.is_contiguous() and abc.shape[-1] == 3
    n = abc.shape[0]
    out = torch.empty_like(abc)
    deg = torch.empty(n, dtype=torch.int32, device=abc.device)
    st = torch.cuda.current_stream(abc.device)
    check(lib().rd_eigen(abc.data_ptr(), n, out.data_ptr(), deg.data_ptr(), C.c_void_p(st.cuda_stream)), "rd_eigen")
    return out, deg


def phase_cycles(det: Detector, on: bool) -> np.ndarray:
    """Read-and-reset the Hough kernel's per-phase cycle counters; enable/disable them."""
    out = np.zeros(16, np.uint64)
    check(lib().rd_phase_cycles(det._h, 1 if on else 0, out.ctypes.data), "rd_phase_cycles")
    return out
