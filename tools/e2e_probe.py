"""H2D bandwidth and end-to-end cfg3 frames/s through the host path for a few chunk sizes:
synchronous Detector.detect_host (RD_HOST_CHUNK: the ramp's largest chunk) and pipelined
submit_host / wait_host with two calls in flight (RD_HOST_CHUNK_PIPE: the chunk behind a call
in flight).  PROBE_CHUNKS / PROBE_PIPE list the sizes."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

if len(sys.argv) > 1:   # child: one chunk size (read at the first host-path call)
    import paper_1310_1371_b200 as rd  # noqa: E402
    import synth  # noqa: E402
    B, K = 256, 10
    fr = torch.from_numpy(synth.batch(3, 0, 0, B)).pin_memory()
    det = rd.Detector(synth.preset(3), max_batch=B)
    outs = [det.detect_host(fr), det.detect_host(fr)]
    if sys.argv[1] == "sync":
        t0 = time.perf_counter()
        for _ in range(K):
            det.detect_host(fr, outs[0])
        tag = f"sync chunk {os.environ.get('RD_HOST_CHUNK', 'default')}"
    else:
        for rep in range(2):   # warm-up, then timed
            t0 = time.perf_counter()
            for i in range(K):
                det.submit_host(fr, outs[i % 2])
                if i:
                    det.wait_host()
            det.wait_host()
        tag = f"pipelined chunk {os.environ.get('RD_HOST_CHUNK_PIPE', 'default')}"
    dt = (time.perf_counter() - t0) / K
    print(f"{tag}: {B / dt:.0f} frames/s ({dt * 1e3:.2f} ms per {B} frames)", flush=True)
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
print(f"H2D pinned: {10 * x.numel() / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
for c in os.environ.get("PROBE_CHUNKS", "48").split():
    subprocess.run([sys.executable, __file__, "sync"], env=dict(os.environ, RD_HOST_CHUNK=c))
for c in os.environ.get("PROBE_PIPE", "48 64 96 128").split():
    subprocess.run([sys.executable, __file__, "pipe"], env=dict(os.environ, RD_HOST_CHUNK_PIPE=c))
