"""NEXT-3: the paper's robustness assessment on the synthetic corpus of
synth/robust.py, scored on the GPU detector's output (ridges, and the NEXT-2 edge variant for
comparison).  The first frames are also run through the oracle and must be identical.

usage: python tools/robustness.py [n_frames=600] [out.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1310_1371_b200 as rd  # noqa: E402
from synth import robust  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
frames, truth = robust.corpus(2026, n)
res = {"corpus": dict(frames=n, size=f"{robust.WIDTH}x{robust.HEIGHT} uint16", seed=2026,
                      paper="PAPER.md:611-627: 600 sub-frames 340x370, 14.3 rings, 67.7 % clustered; "
                            "detection 94.7 %, clustered detection 95.5 %, clustered false 0.8 %")}
for name, params in (("ridges", robust.PARAMS), ("edges", dict(robust.PARAMS, feature=1, edge_threshold=40.0))):
    det = rd.Detector(dict(params, max_entries_per_tile=4096), max_batch=n)
    dev = torch.from_numpy(frames).cuda()
    out = det.detect(dev)
    det.sync()
    t0 = time.perf_counter()
    det.detect(dev, out)
    det.sync()
    dt = time.perf_counter() - t0
    got = out.to_numpy()
    rates, cnt = robust.score(truth, got)
    # parity on the first frames
    k = min(n, 16)
    exp, _ = oracle.detect_batch(oracle.params(**params), frames[:k])
    same = all(len(a) == len(b) and all(np.array_equal(a[f], b[f]) for f in ("cx", "cy", "r", "raw_votes",
               "score_fixed", "inliers", "fit_ok")) for a, b in zip(got[:k], exp))
    res[name] = dict(rates={k2: round(v, 4) for k2, v in rates.items()}, counts=cnt,
                     gpu_frames_per_s=round(n / dt, 1), oracle_identical_first_frames=k if same else 0)
    print(name, json.dumps(res[name]))
if len(sys.argv) > 2:
    json.dump(res, open(sys.argv[2], "w"), indent=1)
