"""Which capacity overflows on the robustness corpus (flags per frame)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1310_1371_b200 as rd
from synth import robust
N = int(os.environ.get("N", "64"))
frames, truth = robust.corpus(2026, N)
extra = dict(a.split("=") for a in sys.argv[1:])
params = dict(robust.PARAMS, max_entries_per_tile=4096)
params.update({k: (float(v) if "." in v else int(v)) for k, v in extra.items()})
det = rd.Detector(params, max_batch=N)
det.detect(torch.from_numpy(frames).cuda())
try:
    det.sync()
except Exception as e:
    print("sync:", e)
fl = det.overflow(N)
print("flags", np.unique(fl, return_counts=True))
