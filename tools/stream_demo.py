"""NEXT-4: streaming ingest at camera-like rates ("70 Hz"; 698-705).

A producer thread "captures" cfg3 frames (1024x688 uint16, 64 distinct frames cycled) at a
target rate into StreamDetector's pinned ring; the consumer detects whatever has arrived.
Reports sustained frames/s and capture->rings latency per rate, and checks that every
streamed frame's rings equal the batch detector's.  usage: stream_demo.py [out.json]"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_1371_b200 as rd  # noqa: E402
from paper_1310_1371_b200.stream import StreamDetector  # noqa: E402
import synth  # noqa: E402

params = synth.preset(3)
src = synth.batch(3, 0, 0, 64)
ref_det = rd.Detector(params, max_batch=64)
ref = ref_det.detect(torch.from_numpy(src).cuda()).to_numpy()
ref_det.sync()
out = {"workload": "cfg3 frames 1024x688 uint16, 64 distinct frames cycled", "runs": []}
for rate, seconds in ((70, 2.0), (1000, 1.0), (5000, 1.0), (0, 1.0)):
    sd = StreamDetector(params, slots=512, max_batch=64)
    lat, ok, batches = [], [True], []
    n_frames = int(rate * seconds) if rate else 20000

    def on_result(i, rings, dt):
        lat.append(dt)
        e = ref[i % 64]
        if len(rings) != len(e) or not all(np.array_equal(rings[k], e[k]) for k in ("cx", "cy", "r", "score_fixed")):
            ok[0] = False

    cons = threading.Thread(target=sd.run, kwargs=dict(on_result=on_result))
    cons.start()
    t0 = time.perf_counter()
    for i in range(n_frames):
        if rate:
            target = t0 + i / rate
            while time.perf_counter() < target:
                time.sleep(max(0.0, min(0.0005, target - time.perf_counter())))
        sd.push(src[i % 64])
        if not rate and time.perf_counter() - t0 > seconds:
            n_frames = i + 1
            break
    sd.close()
    cons.join()
    wall = time.perf_counter() - t0
    lat_ms = np.array(lat) * 1e3
    r = {"target_hz": rate or "unthrottled", "frames": n_frames, "sustained_frames_per_s": round(n_frames / wall, 1),
         "latency_ms_p50": round(float(np.percentile(lat_ms, 50)), 3),
         "latency_ms_p99": round(float(np.percentile(lat_ms, 99)), 3), "latency_ms_max": round(float(lat_ms.max()), 3),
         "rings_equal_batch": ok[0]}
    out["runs"].append(r)
    print(json.dumps(r), flush=True)
    sd.det.close()
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
