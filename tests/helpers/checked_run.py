"""Runs the hot path through librd_checked.so (RD_LIB_PATH) and compares with the oracle.

Invoked by tests/test_checked.py in a subprocess (the library is loaded once per process).
Cases: cfg1, cfg2 batch, cfg3 frames through the byte-counter pass and the forced 16-bit redo
pass, the host path (synchronous and pipelined), the edge variant, and r_max = 100 (K_r >= 16).  Every kernel index is
bounds-checked (RD_CHECKED); rd_sync / rd_detect_host report a failed check as RD_ERR_CUDA.
With RD_JITTER=1 the Hough kernel's warps sleep pseudo-random times at every phase start, so
the shared-memory protocol between phases runs under perturbed schedules.  Prints one line per
case and "checked ok" at the end; exits non-zero on the first difference or failed check.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1310_1371_b200 as rd  # noqa: E402
import synth  # noqa: E402

assert rd._rd.LIB_PATH.endswith("librd_checked.so"), rd._rd.LIB_PATH
INT = ("cx", "cy", "r", "raw_votes", "score_fixed", "inliers", "fit_ok")


def same(got, exp):
    if got is None or len(got) != len(exp):
        return False
    return all(np.array_equal(got[k], exp[k]) for k in INT) and all(
        np.max(np.abs(got[k] - exp[k])) <= 1e-4 for k in ("fx", "fy", "fr", "rms")) if len(exp) else True


def run(name, params, frames, host=False, pipelined=False):
    det = rd.Detector(dict(params, debug=1), max_batch=len(frames) if not pipelined else 4)
    if pipelined:   # three calls, two in flight (rd_submit_host / rd_wait_host), then the middle one
        outs = [det.submit_host(frames), det.submit_host(frames[::-1].copy())]
        det.wait_host()
        outs.append(det.submit_host(frames))
        det.wait_host()
        det.wait_host()
        rev = outs[1].to_numpy()[::-1]
        out = outs[2].to_numpy()
        assert all(a is not None and a.tobytes() == b.tobytes() for a, b in zip(out, rev)), name
    elif host:
        out = det.detect_host(frames).to_numpy()
    else:
        out = det.detect(torch.from_numpy(np.ascontiguousarray(frames)).cuda()).to_numpy()
        det.sync()
    exp, _ = oracle.detect_batch(oracle.params(**params), frames)
    bad = [i for i in range(len(frames)) if not same(out[i], exp[i])]
    print(name, len(frames), "frames", sum(len(e) for e in exp), "rings", "mismatch" if bad else "ok", flush=True)
    if bad:
        sys.exit(3)


run("cfg1", synth.preset(1), np.stack([synth.frame(1, 0, i)[0] for i in range(2)]))
run("cfg2", synth.preset(2), synth.batch(2, 0, 0, 4))
run("cfg3", synth.preset(3), synth.batch(3, 0, 0, 3))
run("cfg3-host", synth.preset(3), synth.batch(3, 0, 10, 5), host=True)
run("cfg2-pipelined", synth.preset(2), synth.batch(2, 0, 20, 9), pipelined=True)
run("cfg2-edges", synth.edge_preset(2), synth.batch(2, 0, 0, 2))
W = H = 320
sc = synth.scene(W, H, pixel_bytes=2, max_value=4095, background=100, sigma_p=1.5, read_sigma=8, poisson=1)
big = np.stack([synth.render(sc, synth.make_rings([(160, 160, 90, 2500), (150, 170, 70, 2000)]), noise_key=k)
                for k in range(2)])
run("r100", dict(width=W, height=H, pixel_bytes=2, max_value=4095, smoothing_sigma=1.5, curvature_threshold=-10.0,
                 r_min=60, r_max=100, vote_threshold_raw=3, vote_threshold_norm=0.5, sig_a=1, sig_b=5, sig_den=20,
                 annulus_halfwidth=0), big)
print("checked ok", flush=True)
