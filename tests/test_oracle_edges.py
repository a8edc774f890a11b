"""Pins of the oracle's directed-edge variant (NEXT-2; -m "not gpu").

PAPER.md:993-997 (SI, Additional notes): "The algorithm is not restricted to directed
ridges as it can be replaced by directed edges ... This is achieved by replacing the
Hessian by the Gradient.  In this case, the gradient magnitude replacing kappa has to be a
local maximum along the gradient direction."  Reading R19 fixes the operator
(OpenCV's 5x5 first-order Sobel, correlation form), the squared-magnitude comparisons and
the threshold units.  The pins use closed forms (linear ramps), brute-force 2D correlation
with a different evaluation order, geometry (edges of a disc lie on its rim and point along
the radius), threshold monotonicity and exact recovery of a disc's centre and radius.
"""
import numpy as np

import oracle
import synth

S5 = np.array([1, 4, 6, 4, 1], dtype=np.float64)
D1 = np.array([-1, -2, 0, 2, 1], dtype=np.float64)


def P(**kw):
    base = dict(width=64, height=64, pixel_bytes=2, smoothing_sigma=1.5, curvature_threshold=-10.0, r_min=8,
                r_max=30, vote_threshold_raw=3, vote_threshold_norm=0.5, sig_a=1, sig_b=5, sig_den=20,
                annulus_halfwidth=0, feature=1, edge_threshold=20.0)
    base.update(kw)
    return oracle.params(**base)


def disc(W, H, cx, cy, R, amp=1000.0, bg=100.0, width=1.0):
    yy, xx = np.mgrid[0:H, 0:W]
    d = np.hypot(xx - cx, yy - cy)
    return np.clip(np.rint(bg + amp / (1.0 + np.exp((d - R) / width))), 0, 4095).astype(np.uint16)


def test_gradient_of_ramp_closed_form():
    """I = a x + b y + c: the unnormalised smoothing multiplies a linear image by (sum q)^2,
    d1 = [-1,-2,0,2,1] has gain 8 on x and s5 gain 16, so Ix = 128 (sum q)^2 a and
    Iy = 128 (sum q)^2 b away from the border."""
    p = P(width=48, height=40)
    a, b = 7, 3
    yy, xx = np.mgrid[0:40, 0:48]
    img = (a * xx + b * yy + 100).astype(np.uint16)
    Ix, Iy = oracle.gradient(p, oracle.smooth(p, img))
    sq = int(oracle.gauss_taps(1.5).sum())
    m = 5 + 2 + 1   # K_s + Sobel reach + 1: the replicate border does not reach the interior
    assert np.all(Ix[m:-m, m:-m] == 128 * sq * sq * a)
    assert np.all(Iy[m:-m, m:-m] == 128 * sq * sq * b)


def test_gradient_brute_force_2d_correlation():
    """The separable passes equal the 2D correlation with s5 (x) d1 (Ix) and d1 (x) s5 (Iy)
    on [2,W-3]x[2,H-3] (different evaluation order, exact integers)."""
    rng = np.random.default_rng(5)
    p = P(width=17, height=15)
    G = rng.integers(-10 ** 6, 10 ** 6, size=(15, 17)).astype(np.float64)
    Ix, Iy = oracle.gradient(p, G)
    kx, ky = np.outer(S5, D1), np.outer(D1, S5)
    for y in range(2, 15 - 2):
        for x in range(2, 17 - 2):
            win = G[y - 2:y + 3, x - 2:x + 3]
            assert Ix[y, x] == (kx * win).sum()
            assert Iy[y, x] == (ky * win).sum()
    assert not Ix[:2].any() and not Iy[:, :2].any()


def test_constant_frame_has_no_edges():
    p = P()
    assert len(oracle.ridges(p, np.full((64, 64), 700, np.uint16))) == 0


def test_disc_edges_on_rim_and_radial():
    """Edges of a bright disc are the maxima of |grad| across the rim: within 1 px of R,
    with the gradient pointing to the centre (toward the brighter side) within 0.15 rad."""
    cx, cy, R = 31, 29, 17.3
    p = P()
    E = oracle.ridges(p, disc(64, 64, cx, cy, R))
    assert len(E) > 0.8 * 2 * np.pi * R
    d = np.hypot(E["x"] - cx, E["y"] - cy)
    assert np.all(np.abs(d - R) <= 1.0)
    cosang = -((E["x"] - cx) * E["dx"] + (E["y"] - cy) * E["dy"]) / d
    assert np.all(cosang >= np.cos(0.15))
    assert np.allclose(E["dx"] ** 2 + E["dy"] ** 2, 1.0, atol=1e-14)


def test_edge_threshold_monotone():
    """The local-maximum test does not depend on the threshold, so raising it removes
    edges and never adds any; a threshold above the steepest flank leaves none."""
    img = synth.batch(1, 0, 0, 1)[0]
    base = synth.edge_preset(1)
    sets = []
    for t in (2.0, 10.0, 40.0):
        E = oracle.ridges(oracle.params(**dict(base, edge_threshold=t)), img)
        sets.append({(int(e["x"]), int(e["y"])) for e in E})
    assert sets[1] <= sets[0] and sets[2] <= sets[1] and len(sets[2]) < len(sets[0])
    assert len(oracle.ridges(oracle.params(**dict(base, edge_threshold=1e6)), img)) == 0


def test_edge_translation_equivariance():
    """Shifting the frame content by (dx, dy) away from the border shifts the edge set."""
    p = P()
    a = oracle.ridges(p, disc(64, 64, 30, 31, 14.6))
    b = oracle.ridges(p, disc(64, 64, 33, 29, 14.6))
    assert {(int(e["x"]) + 3, int(e["y"]) - 2) for e in a} == {(int(e["x"]), int(e["y"])) for e in b}


def test_edge_detection_recovers_disc_exactly():
    """A noiseless disc with integer centre and radius yields exactly one peak, at its
    centre and radius, supported by all of its edges."""
    for (cx, cy, R) in ((40, 38, 12), (44, 41, 20), (41, 43, 27)):
        p = P(width=84, height=84)
        img = disc(84, 84, cx, cy, float(R))
        rings, st = oracle.detect(p, img)
        assert len(rings) == 1, (R, rings)
        r = rings[0]
        assert (int(r["cx"]), int(r["cy"]), int(r["r"])) == (cx, cy, R)
        assert r["inliers"] == st["ridges"]
        assert abs(r["fx"] - cx) < 0.05 and abs(r["fy"] - cy) < 0.05 and abs(r["fr"] - R) < 0.5


def test_streamed_method_equals_full_array_on_edges():
    """The paper's streamed Hough stage (oracle/streamed.c) reaches the full-array result
    with edges as well (it only consumes the feature list)."""
    params = synth.edge_preset(2)
    frames = synth.batch(2, 0, 0, 2)
    p = oracle.params(**params)
    a = oracle.detect_batch(p, frames, streamed=False)
    b = oracle.detect_batch(p, frames, streamed=True)
    for x, y in zip(a[0], b[0]):
        assert np.array_equal(x, y)
