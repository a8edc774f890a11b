"""B200-native ridge-directed circle-Hough ring detector (Afik, arXiv 1310.1371).

The detection path runs entirely in the sm_100a CUDA kernels of csrc/ behind the C ABI
of include/rd.h (librd.so).  This package is a thin binding: PyTorch supplies device
memory, streams and process groups only.
"""
from ._rd import FPR_DTYPE, HOT_DTYPE, RIDGE_DTYPE, RING_DTYPE, STATS_DTYPE, RDError, lib  # noqa: F401
from .detector import Detector, RingBatch, eigen  # noqa: F401

__all__ = ["Detector", "RingBatch", "eigen", "RING_DTYPE", "RIDGE_DTYPE", "HOT_DTYPE", "STATS_DTYPE", "FPR_DTYPE",
           "RDError", "lib"]
