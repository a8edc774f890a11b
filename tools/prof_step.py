"""Small fixed workload for ncu captures: cfg3 frames, a few rd_detect calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_1371_b200 as rd  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 3
params = synth.preset(cfg)
frames = torch.from_numpy(synth.batch(cfg, 0, 0, B)).cuda()
det = rd.Detector(params, max_batch=B)
for _ in range(calls):
    out = det.detect(frames)
det.sync()
print("ok", int(out.counts.sum()))
