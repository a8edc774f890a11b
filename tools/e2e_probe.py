"""H2D bandwidth and end-to-end frames/s of Detector.detect_host for a few host chunk sizes."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

if len(sys.argv) > 1:   # child: one chunk size (RD_HOST_CHUNK is read at the first detect_host)
    import paper_1310_1371_b200 as rd  # noqa: E402
    import synth  # noqa: E402
    B = 256
    fr = torch.from_numpy(synth.batch(3, 0, 0, B)).pin_memory()
    det = rd.Detector(synth.preset(3), max_batch=B)
    out = det.detect_host(fr)
    det.detect_host(fr, out)
    t0 = time.perf_counter()
    for _ in range(5):
        det.detect_host(fr, out)
    dt = (time.perf_counter() - t0) / 5
    print(f"chunk {os.environ.get('RD_HOST_CHUNK')}: {B / dt:.0f} frames/s ({dt * 1e3:.2f} ms per 256 frames)")
    sys.exit(0)
x = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(3):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D pinned: {10 * x.numel() / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
for c in os.environ.get("PROBE_CHUNKS", "16 32 48 64 96 128").split():
    subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, RD_HOST_CHUNK=c))
