"""NEXT-3: the robustness corpus (synth/robust.py) and its scorer (-m "not gpu").

PAPER.md:611-627: 600 sub-frames of 340 x 370 px, 14.3 rings per sub-frame, 67.7 % in
clusters (overlap and inclusion); detection 94.7 %, clustered detection 95.5 %, clustered
false 0.8 %.  These tests pin the corpus to that shape, the scorer to hand-made cases, and
the oracle's quality on it (the GPU path must reproduce the oracle's rings; tests/
test_gpu_parity.py and tools/robustness.py).
"""
import numpy as np

import oracle
from synth import robust


def test_corpus_shape_matches_paper():
    frames, truth = robust.corpus(11, 200)
    assert frames.shape == (200, 370, 340) and frames.dtype == np.uint16
    n = np.array([len(r) for r, _ in truth])
    cl = sum(int(c.sum()) for _, c in truth) / n.sum()
    assert set(n) <= {14, 15} and 14.15 <= n.mean() <= 14.45
    assert 0.63 <= cl <= 0.72


def test_corpus_clusters_overlap_or_nest_and_singles_are_isolated():
    for i in range(50):
        rings, cl = robust.layout(3, i)
        x, y, r = rings["cx"], rings["cy"], rings["r"]
        for a in range(len(r)):
            d = np.hypot(x - x[a], y - y[a])
            touching = [(b, d[b]) for b in range(len(r)) if b != a and d[b] < r[a] + r[b] + 3 * robust.SIGMA_P + 2]
            if cl[a]:
                assert any(dd < r[a] + r[b] for b, dd in touching)   # its partner overlaps or contains it
            else:
                assert not touching


def test_scorer_hand_cases():
    rings, cl = robust.layout(5, 0)
    det = np.zeros(len(rings), dtype=[("fx", "f8"), ("fy", "f8"), ("fr", "f8")])
    det["fx"], det["fy"], det["fr"] = rings["cx"], rings["cy"], rings["r"]
    rates, _ = robust.score([(rings, cl)], [det])
    assert rates["detection_rate"] == 1.0 and rates["false_rate"] == 0.0
    rates, c = robust.score([(rings, cl)], [det[1:]])
    assert c["found"] == len(rings) - 1 and c["false"] == 0
    fake = det[:1].copy()
    fake["fr"] += 5.0                       # radius off by more than the tolerance
    rates, c = robust.score([(rings, cl)], [np.concatenate([det, fake])])
    assert c["found"] == len(rings) and c["false"] == 1


def test_oracle_quality_on_corpus():
    """The method (oracle) finds most rings of the synthetic corpus and reports few false
    ones: detection and clustered-detection rates above 90 %, false rate below 5 %."""
    frames, truth = robust.corpus(2026, 24)
    dets, _ = oracle.detect_batch(oracle.params(**robust.PARAMS), frames)
    rates, _ = robust.score(truth, dets)
    assert rates["detection_rate"] > 0.9 and rates["clustered_detection_rate"] > 0.9
    assert rates["false_rate"] < 0.05
