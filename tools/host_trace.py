import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1310_1371_b200 as rd
import synth
B = 256
fr = torch.from_numpy(synth.batch(3, 0, 0, B)).pin_memory()
det = rd.Detector(synth.preset(3), max_batch=B)
hr = torch.empty((B, det.ring_cap, 64), dtype=torch.uint8).pin_memory()
hc = torch.empty((B,), dtype=torch.int32).pin_memory()
for _ in range(3):
    det.detect_host(fr, hr, hc)
os.environ["RD_HOST_TRACE"] = "1"
t0 = time.perf_counter()
det.detect_host(fr, hr, hc)
print("wall ms", (time.perf_counter() - t0) * 1e3)
