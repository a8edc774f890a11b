"""NEXT-1: the paper's streamed Hough stage equals the full-array definition.

PAPER.md:402-434 says the vote stack, the 3-level sub-spaces indexed by r mod 3 and the
register-and-undo bookkeeping change memory and speed, not results; SI steps 2-4
 give the procedure.  oracle/streamed.c follows those steps; here it
must reproduce orc_peaks on the full [N_r, H, W] accumulator hotspot for hotspot and peak
for peak (same values, same canonical order), on the synthetic configs and on adversarial
ridge lists (low thresholds, many ties, votes at every border).
"""
import numpy as np
import pytest

import oracle
import synth


def _full(p, rid):
    raw, _ = oracle.votes(p, rid)
    return oracle.peaks(p, raw)


def _same(a, b):
    assert len(a) == len(b)
    for f in ("r", "y", "x", "raw", "S"):
        assert np.array_equal(a[f], b[f]), f


@pytest.mark.parametrize("cfg,idx", [(1, 0), (1, 5), (11, 2), (2, 0), (2, 7), (3, 0)])
def test_streamed_equals_full_array_on_configs(cfg, idx):
    p = oracle.params(**synth.preset(cfg))
    img, _ = synth.frame(cfg, 0, idx)
    rid = oracle.ridges(p, img)
    pk_s, hot_s = oracle.stream_peaks(p, rid)
    pk_f, hot_f = _full(p, rid)
    _same(hot_s, hot_f)
    _same(pk_s, pk_f)
    assert len(pk_s) > 0
    rings, st, _, hot_d = oracle.detect(p, img, want_debug=True)
    _same(hot_s, hot_d)
    assert st["peaks"] == len(pk_s)


def _random_ridges(rng, W, H, n, integer_dirs):
    rid = np.zeros(n, dtype=oracle.RIDGE_DTYPE)
    rid["x"] = rng.integers(0, W, n)
    rid["y"] = rng.integers(0, H, n)
    if integer_dirs:   # axis/diagonal directions: exact plateaus and ties in S
        d = np.array([(1, 0), (0, 1), (-1, 0), (0, -1), (1, 1), (1, -1)], dtype=np.float64)
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        k = rng.integers(0, len(d), n)
        rid["dx"], rid["dy"] = d[k, 0], d[k, 1]
    else:
        a = rng.uniform(0, 2 * np.pi, n)
        rid["dx"], rid["dy"] = np.cos(a), np.sin(a)
    order = np.lexsort((rid["x"], rid["y"]))
    return rid[order]


@pytest.mark.parametrize("seed", range(8))
def test_streamed_equals_full_array_adversarial(seed):
    rng = np.random.default_rng(1000 + seed)
    W, H = int(rng.integers(12, 40)), int(rng.integers(12, 40))
    p = oracle.params(width=W, height=H, pixel_bytes=2, smoothing_sigma=1.0, curvature_threshold=-4.0,
                      r_min=int(rng.integers(1, 4)), r_max=int(rng.integers(5, 14)),
                      vote_threshold_raw=int(rng.integers(0, 3)), vote_threshold_norm=float(rng.choice([0.0, 0.05])),
                      sig_a=1, sig_b=5, sig_den=20, annulus_halfwidth=0)
    rid = _random_ridges(rng, W, H, int(rng.integers(20, 400)), integer_dirs=bool(seed % 2))
    pk_s, hot_s = oracle.stream_peaks(p, rid)
    pk_f, hot_f = _full(p, rid)
    _same(hot_s, hot_f)
    _same(pk_s, pk_f)


def test_streamed_empty_and_single_level():
    p = oracle.params(width=16, height=16, pixel_bytes=2, smoothing_sigma=1.0, curvature_threshold=-4.0, r_min=3,
                      r_max=3, vote_threshold_raw=0, vote_threshold_norm=0.0, sig_a=1, sig_b=5, sig_den=20,
                      annulus_halfwidth=0)
    pk, hot = oracle.stream_peaks(p, np.zeros(0, dtype=oracle.RIDGE_DTYPE))
    assert len(pk) == 0 and len(hot) == 0
    rid = _random_ridges(np.random.default_rng(7), 16, 16, 60, integer_dirs=True)
    pk_s, hot_s = oracle.stream_peaks(p, rid)
    pk_f, hot_f = _full(p, rid)
    _same(hot_s, hot_f)
    _same(pk_s, pk_f)


@pytest.mark.parametrize("cfg", [2, 3])
def test_streamed_batch_rings_identical(cfg):
    """Whole pipeline with the streamed stage: byte-identical rings and stats, threads reusing
    their workspace across frames (the undo must leave it zero)."""
    p = oracle.params(**synth.preset(cfg))
    frames = synth.batch(cfg, 0, 0, 4 if cfg == 3 else 6)
    r_full, st_full = oracle.detect_batch(p, frames, nthreads=2)
    r_str, st_str = oracle.detect_batch(p, frames, nthreads=2, streamed=True)
    for a, b in zip(r_full, r_str):
        assert a.tobytes() == b.tobytes()
    assert st_full.tobytes() == st_str.tobytes()
