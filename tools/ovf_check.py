"""Which frames of a cfg3 batch overflow a device capacity (flags per frame); HC/EC override the caps."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1310_1371_b200 as rd, synth
B = 128
params = dict(synth.preset(3), max_hotspots_per_level=int(os.environ.get("HC", 0)), max_entries_per_tile=int(os.environ.get("EC", 0)))
frames = torch.from_numpy(synth.batch(3, 0, 0, B)).cuda()
det = rd.Detector(params, max_batch=B)
rings, counts = det.detect(frames)
det.sync(raise_on_overflow=False)
ovf = det.overflow(B)
print("overflow flags:", {i: int(v) for i, v in enumerate(ovf) if v})
