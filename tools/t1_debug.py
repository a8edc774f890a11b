"""Debug helper: run rd_detect over a few (pixel type, size, sigma) combinations, one process each."""
import sys
import subprocess

sys.path.insert(0, '/root/repo')
if len(sys.argv) > 1:
    import numpy as np
    import torch
    import paper_1310_1371_b200 as rd
    pb, W, H, sig = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
    params = dict(width=W, height=H, pixel_bytes=pb, max_value=255 if pb == 1 else 4095, smoothing_sigma=sig,
                  curvature_threshold=-4.0, r_min=5, r_max=30)
    frames = np.random.default_rng(0).integers(0, 200, (2, H, W)).astype(np.uint8 if pb == 1 else np.uint16)
    det = rd.Detector(params, max_batch=2)
    try:
        r, c = det.detect(torch.from_numpy(frames).cuda())
        det.sync()
        print(sys.argv[1:], "ok", c.tolist(), flush=True)
    except Exception as e:
        print(sys.argv[1:], "ERR", str(e)[:120], flush=True)
else:
    for args in (["2", "128", "128", "1.0"], ["2", "128", "128", "1.5"], ["1", "128", "128", "1.5"], ["1", "640", "480", "1.2"],
                 ["1", "640", "480", "1.5"], ["2", "640", "480", "1.2"], ["1", "128", "128", "1.0"]):
        subprocess.run([sys.executable, __file__] + args, env={**__import__("os").environ, "CUDA_LAUNCH_BLOCKING": "1"})
