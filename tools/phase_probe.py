"""Per-phase cycle breakdown of the Hough kernel and per-kernel event times.

usage: phase_probe.py [cfg] [batch]   (env: RD_K2_SHAPE=T,G,threads,ctas  PROBE_ENTRY_CAP=n  PROBE_HOT_CAP=n)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_1371_b200 as rd  # noqa: E402
from paper_1310_1371_b200.detector import phase_cycles  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
params = synth.preset(cfg)
if os.environ.get("PROBE_ENTRY_CAP"):
    params["max_entries_per_tile"] = int(os.environ["PROBE_ENTRY_CAP"])
if os.environ.get("PROBE_HOT_CAP"):
    params["max_hotspots_per_level"] = int(os.environ["PROBE_HOT_CAP"])
frames = torch.from_numpy(synth.batch(cfg, 0, 0, B)).cuda()
det = rd.Detector(params, max_batch=B)
for _ in range(2):
    det.detect(frames)
st = det.sync(raise_on_overflow=False)
ovf = det.flags(B)
det.set_timing(True)
for _ in range(3):
    det.detect(frames)
det.sync(raise_on_overflow=False)
ms, n = det.kernel_times()
print("shape", os.environ.get("RD_K2_SHAPE", "default"), "overflow frames", int((ovf != 0).sum()),
      "kernel us/frame:", [round(1000 * m / n / B, 2) for m in ms])
det.set_timing(False)
phase_cycles(det, True)
det.detect(frames)
det.sync(raise_on_overflow=False)
c = phase_cycles(det, False)
names = ["rays", "setup0", "votes", "S", "cand+undo", "nms+setup"]
ncta = int(c[15])
tot = sum(int(x) for x in c[:6])
print("  CTAs", ncta, "cycles/CTA", round(tot / max(ncta, 1)), " ".join(
    f"{nm}={int(c[i]) / max(ncta, 1):.0f}" for i, nm in enumerate(names)))
