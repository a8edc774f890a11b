"""Capacities a config needs (rd_query_overflow) and per-kernel us/frame: usage cap_probe.py cfg n [key=val ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_1371_b200 as rd  # noqa: E402
import synth  # noqa: E402

cfg, n = int(sys.argv[1]), int(sys.argv[2])
params = synth.preset(cfg)
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    params[k] = int(v)
frames = torch.from_numpy(synth.batch(cfg, 0, 0, n)).cuda()
det = rd.Detector(params, max_batch=n)
det.detect(frames)
det.sync(raise_on_overflow=False)
print("overflow", det.overflow())
det.set_timing(True)
for _ in range(3):
    det.detect(frames)
ms, calls = det.kernel_times()
print("us/frame K1 K1.5 K2 K3:", [round(1000 * m / calls / n, 2) for m in ms])
