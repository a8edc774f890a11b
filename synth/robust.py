"""NEXT-3 robustness corpus: seeded synthetic sub-frames shaped like the paper's assessment set.

PAPER.md:611-627 ("Robustness assessment"): 600 sub-frames of 340 x 370 px from the chaotic-
flow experiment, 14.3 rings per sub-frame on average, 67.7 % of them in ring clusters
(overlap and inclusion configurations); the paper reports a detection rate of 94.7 % (6.8 %
false negatives before excluding two wall artefacts), 95.5 % of the clustered rings found
and 0.8 % of the reported clustered rings non-existing.  The paper's frames are not
available, so this module generates frames with known truth in the same shape: 14 or 15
rings (mean 14.3), about two thirds of them in overlapping or nested pairs, cfg3 intensities
(12-bit, crest 800-3000 on 100, Poisson + read noise 8, profile sigma 1.5).  It holds no
method arithmetic: layout and rendering only (rendering is synth.render).
"""
from __future__ import annotations

import numpy as np

from . import make_rings, render, scene

WIDTH, HEIGHT = 340, 370
R_LO, R_HI = 10.0, 40.0
SIGMA_P = 1.5
PARAMS = dict(width=WIDTH, height=HEIGHT, pixel_bytes=2, max_value=4095, smoothing_sigma=1.5,
              curvature_threshold=-10.0, r_min=8, r_max=45, vote_threshold_raw=3, vote_threshold_norm=0.5,
              sig_a=1, sig_b=5, sig_den=20, annulus_halfwidth=0, feature=0, edge_threshold=0.0)


def _fits(x, y, r):
    m = r + 3 * SIGMA_P + 3
    return m <= x <= WIDTH - 1 - m and m <= y <= HEIGHT - 1 - m


def layout(seed: int, idx: int):
    """Rings (RING_DTYPE) of sub-frame idx and a per-ring 'clustered' flag."""
    rng = np.random.default_rng([0x6E787433, seed, idx])
    n = 15 if rng.random() < 0.3 else 14                      # mean 14.3
    n_cl = 2 * int(0.677 * n / 2 + rng.random())              # rings in overlap / nested pairs (E = 67.7 %)
    rings, clustered = [], []

    def clear_of_all(x, y, r, skip=()):
        for k, (xo, yo, ro, _) in enumerate(rings):
            if k in skip:
                continue
            if np.hypot(x - xo, y - yo) < r + ro + 3 * SIGMA_P + 2:
                return False
        return True

    tries = 0
    while len(rings) < n_cl and tries < 20000:
        tries += 1
        r1 = rng.uniform(R_LO, R_HI)
        x1, y1 = rng.uniform(0, WIDTH), rng.uniform(0, HEIGHT)
        if rng.random() < 0.7:   # overlap: annuli intersect, |r1 - r2| < d < r1 + r2
            r2 = rng.uniform(R_LO, R_HI)
            d = rng.uniform(abs(r1 - r2) + 4, r1 + r2 - 4) if r1 + r2 - 4 > abs(r1 - r2) + 4 else None
        else:                     # inclusion: nested, d < |r1 - r2| - 4
            r2 = rng.uniform(max(R_LO, r1 * 0.35), r1 - 6) if r1 - 6 > max(R_LO, r1 * 0.35) else None
            d = rng.uniform(0, max(0.0, r1 - r2 - 4)) if r2 is not None else None
        if d is None or r2 is None:
            continue
        a = rng.uniform(0, 2 * np.pi)
        x2, y2 = x1 + d * np.cos(a), y1 + d * np.sin(a)
        if not (_fits(x1, y1, r1) and _fits(x2, y2, r2)):
            continue
        if not (clear_of_all(x1, y1, r1) and clear_of_all(x2, y2, r2)):
            continue
        for (x, y, r) in ((x1, y1, r1), (x2, y2, r2)):
            rings.append((x, y, r, rng.uniform(700, 2900)))
            clustered.append(True)
    while len(rings) < n and tries < 40000:
        tries += 1
        r = rng.uniform(R_LO, R_HI)
        x, y = rng.uniform(0, WIDTH), rng.uniform(0, HEIGHT)
        if _fits(x, y, r) and clear_of_all(x, y, r):
            rings.append((x, y, r, rng.uniform(700, 2900)))
            clustered.append(False)
    return make_rings(rings), np.array(clustered, dtype=bool)


def frame(seed: int, idx: int):
    """(image uint16 [370, 340], truth rings, clustered flags)."""
    rings, cl = layout(seed, idx)
    sc = scene(WIDTH, HEIGHT, pixel_bytes=2, max_value=4095, background=100.0, sigma_p=SIGMA_P, read_sigma=8.0,
               poisson=1)
    img = render(sc, rings, noise_key=(seed << 32) ^ (0x5EED0000 + idx))
    return img, rings, cl


def corpus(seed: int, n: int):
    frames = np.empty((n, HEIGHT, WIDTH), dtype=np.uint16)
    truth = []
    for i in range(n):
        frames[i], rings, cl = frame(seed, i)
        truth.append((rings, cl))
    return frames, truth


def score(truth, detections, centre_tol=2.0, radius_tol=2.0):
    """Match detections (arrays with fx, fy, fr) to truth one-to-one (greedy by distance):
    a pair matches if the centres are within max(centre_tol, 0.1 r) and the radii within
    radius_tol.  A detection is 'in a cluster' if its circle intersects or contains another
    detection's circle.  Returns the counts behind the paper's four rates."""
    c = dict(truth=0, found=0, truth_cl=0, found_cl=0, det=0, false=0, det_cl=0, false_cl=0)
    for (rings, cl), det in zip(truth, detections):
        tx, ty, tr = rings["cx"], rings["cy"], rings["r"]
        dx, dy, dr = (np.asarray(det[k], dtype=np.float64) for k in ("fx", "fy", "fr"))
        pairs = []
        for i in range(len(tx)):
            for j in range(len(dx)):
                dc = np.hypot(tx[i] - dx[j], ty[i] - dy[j])
                if dc <= max(centre_tol, 0.1 * tr[i]) and abs(tr[i] - dr[j]) <= radius_tol:
                    pairs.append((dc + abs(tr[i] - dr[j]), i, j))
        used_t, used_d = set(), set()
        for _, i, j in sorted(pairs):
            if i not in used_t and j not in used_d:
                used_t.add(i)
                used_d.add(j)
        det_cl = np.zeros(len(dx), dtype=bool)
        for j in range(len(dx)):
            for k in range(len(dx)):
                if j != k and np.hypot(dx[j] - dx[k], dy[j] - dy[k]) < dr[j] + dr[k]:
                    det_cl[j] = True
        c["truth"] += len(tx)
        c["found"] += len(used_t)
        c["truth_cl"] += int(cl.sum())
        c["found_cl"] += sum(1 for i in used_t if cl[i])
        c["det"] += len(dx)
        c["false"] += len(dx) - len(used_d)
        c["det_cl"] += int(det_cl.sum())
        c["false_cl"] += sum(1 for j in range(len(dx)) if det_cl[j] and j not in used_d)
    rates = dict(detection_rate=c["found"] / max(1, c["truth"]),
                 clustered_detection_rate=c["found_cl"] / max(1, c["truth_cl"]),
                 false_rate=c["false"] / max(1, c["det"]),
                 clustered_false_rate=c["false_cl"] / max(1, c["det_cl"]),
                 rings_per_frame=c["truth"] / max(1, len(truth)),
                 clustered_fraction=c["truth_cl"] / max(1, c["truth"]))
    return rates, c
