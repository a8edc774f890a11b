"""StreamDetector: frames arriving one at a time (a camera), rings out as soon as possible.

NEXT-4: the paper's real-time use case — 3d tracking "at 70 Hz" on a
desktop with frames handed to worker processes as they are
captured.  Frames are written by the producer into a ring of pinned host
slots; the consumer takes every frame that has arrived (up to max_batch, never waiting for
more) and runs them through rd_detect_host, whose host->device copies overlap the kernels.
So at low rates each frame is detected alone (lowest latency) and at high rates batches grow
until the GPU keeps up.  Only argument marshalling happens here; detection is the C ABI.
"""
from __future__ import annotations

import threading
import time

import numpy as np
import torch

from ._rd import RING_DTYPE
from .detector import Detector, RingBatch


class StreamDetector:
    def __init__(self, params: dict, slots: int = 256, max_batch: int = 64, device: int = 0):
        self.det = Detector(params, max_batch=max_batch, device=device)
        self.max_batch = max_batch
        H, W = int(params["height"]), int(params["width"])
        dt = torch.uint8 if int(params["pixel_bytes"]) == 1 else torch.uint16
        self.slots = slots
        self.frames = torch.empty((slots, H, W), dtype=dt).pin_memory()
        cap = max_batch * self.det.ring_cap   # one batch's compact output, reused
        self.out = RingBatch(np.empty(cap, dtype=RING_DTYPE), np.empty(max_batch, dtype=np.int32),
                             np.empty(max_batch + 1, dtype=np.int32))
        self.t_capture = np.zeros(slots)
        self._written = 0        # frames captured so far
        self._done = 0           # frames detected so far
        self._cv = threading.Condition()
        self.closed = False

    def push(self, frame: np.ndarray) -> int:
        """Producer side: copy one frame into the next slot (blocks while the ring is full)."""
        with self._cv:
            while self._written - self._done >= self.slots:
                self._cv.wait()
            i = self._written % self.slots
        self.frames[i].numpy()[...] = frame
        with self._cv:
            self.t_capture[i] = time.perf_counter()
            self._written += 1
            self._cv.notify_all()
            return self._written - 1

    def close(self):
        with self._cv:
            self.closed = True
            self._cv.notify_all()

    def run(self, on_result=None):
        """Consumer loop until close(): detect every frame that has arrived (contiguous slots,
        up to max_batch), then report (frame index, rings, latency seconds) per frame."""
        while True:
            with self._cv:
                while self._written == self._done and not self.closed:
                    self._cv.wait()
                if self._written == self._done and self.closed:
                    return
                first, avail = self._done, self._written - self._done
            i0 = first % self.slots
            n = min(avail, self.max_batch, self.slots - i0)   # contiguous in the ring
            out = self.det.detect_host(self.frames[i0:i0 + n], self.out)
            t = time.perf_counter()
            if on_result is not None:
                for k in range(n):
                    c, o = int(out.counts[k]), int(out.offsets[k])
                    on_result(first + k, out.rings[o:o + max(c, 0)].copy(), t - self.t_capture[i0 + k])
            with self._cv:
                self._done += n
                self._cv.notify_all()
