"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the PAPER.md passage (or the mathematical fact) it pins.  None of
them re-types the oracle's own formula: they use closed forms, brute force on tiny
inputs with a different evaluation order, library routines (numpy eigh), values
printed in the paper (tests/golden/paper_values.json) and geometric invariants.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def P(**kw):
    base = dict(width=48, height=48, pixel_bytes=2, smoothing_sigma=1.5, curvature_threshold=-10.0, r_min=5,
                r_max=30, vote_threshold_raw=3, vote_threshold_norm=0.5, sig_a=1, sig_b=5, sig_den=20,
                annulus_halfwidth=0)
    base.update(kw)
    return oracle.params(**base)


# ------------------------------------------------------------------ sigma(r), tables
def test_sigma_of_r_paper_values():
    """sigma(r) = 0.05 r + 0.25 (golden points)."""
    p = P()
    for r, s in GOLDEN["sigma_of_r"]["points"]:
        assert oracle.sigma(p, r) == pytest.approx(s, abs=1e-12)


def test_level_halfwidth_is_three_sigma():
    """K_r = ceil(3 sigma(r)) from the golden sigma values (reading R12)."""
    p = P()
    for r, s in GOLDEN["sigma_of_r"]["points"]:
        if r >= 2:
            assert oracle.level_halfwidth(p, r) == math.ceil(3 * s - 1e-12)


@pytest.mark.parametrize("r", [10, 20, 35, 55, 71, 91])
def test_level_weights_are_gaussian_of_width_sigma_r(r):
    """The weights are a sampled Gaussian of width sigma(r): peak 2^12, symmetric
    decay, and second moment ~ sigma(r)^2 (a 3-sigma truncated Gaussian keeps 0.973 sigma^2)."""
    p = P()
    K = oracle.level_halfwidth(p, r)
    w = np.array([oracle.level_weight(p, r, abs(d)) for d in range(-K, K + 1)], dtype=np.float64)
    d = np.arange(-K, K + 1)
    assert w[K] == 4096
    assert np.all(np.diff(w[K:]) < 0)
    var = float((d * d * w).sum() / w.sum())
    s = 0.05 * r + 0.25
    assert 0.90 * s * s <= var <= 1.05 * s * s


@pytest.mark.parametrize("sig", [1.0, 1.2, 1.5, 2.0])
def test_gauss_taps_shape(sig):
    """Smoothing taps: centre 2^10, symmetric, support ceil(3 sigma),
    second moment ~ sigma^2."""
    q = oracle.gauss_taps(sig).astype(np.float64)
    K = (len(q) - 1) // 2
    assert K == math.ceil(3 * sig)
    assert q[K] == 1024 and np.array_equal(q, q[::-1])
    d = np.arange(-K, K + 1)
    var = float((d * d * q).sum() / q.sum())
    assert 0.9 * sig * sig <= var <= 1.05 * sig * sig


def test_norm_threshold_is_tau_two_pi():
    """Candidate threshold: N = S/(2^24 r) > tau * 2 pi."""
    p = P(vote_threshold_norm=0.5)
    for r in (5, 17, 30):
        assert oracle.norm_threshold(p, r) / (2 ** 24 * r) == pytest.approx(0.5 * 2 * math.pi, rel=1e-15)


# ------------------------------------------------------------------ step 1: smoothing
def _brute_smooth(img, q):
    K = (len(q) - 1) // 2
    pad = np.pad(img.astype(np.int64), K, mode="edge")
    H, W = img.shape
    G = np.zeros((H, W), dtype=np.int64)
    for i in range(-K, K + 1):
        for j in range(-K, K + 1):
            G += int(q[i + K]) * int(q[j + K]) * pad[K + i:K + i + H, K + j:K + j + W]
    return G


def test_smooth_constant_and_impulse():
    """A constant image stays constant (x (sum q)^2); an impulse reproduces the 2D kernel q q^T."""
    p = P(width=24, height=20)
    q = oracle.gauss_taps(1.5).astype(np.int64)
    G = oracle.smooth(p, np.full((20, 24), 777, np.uint16))
    assert np.all(G == 777 * q.sum() ** 2)
    img = np.zeros((20, 24), np.uint16)
    img[10, 12] = 1
    G = oracle.smooth(p, img)
    K = (len(q) - 1) // 2
    assert np.array_equal(G[10 - K:10 + K + 1, 12 - K:12 + K + 1], np.outer(q, q).astype(np.float64))


@pytest.mark.parametrize("seed", range(3))
def test_smooth_matches_brute_force_2d(seed):
    """Separable evaluation == direct 2D sum with replicate border, exactly."""
    rng = np.random.default_rng(seed)
    for pb, sig in ((1, 1.0), (2, 1.5), (2, 1.2)):
        img = rng.integers(0, 256 if pb == 1 else 65536, size=(17, 23)).astype(np.uint8 if pb == 1 else np.uint16)
        p = P(width=23, height=17, pixel_bytes=pb, smoothing_sigma=sig)
        G = oracle.smooth(p, img)
        assert np.array_equal(G, _brute_smooth(img, oracle.gauss_taps(sig)).astype(np.float64))


# ------------------------------------------------------------------ step 2: Hessian
S5 = np.array([1, 4, 6, 4, 1])
D2 = np.array([1, 0, -2, 0, 1])
D1 = np.array([-1, -2, 0, 2, 1])


def _interior(p, K):
    m = K + 2
    return slice(m, p.height - m), slice(m, p.width - m)


def test_hessian_polynomials():
    """Exact polynomial identities of the 5x5 second-order Sobel on smoothed quadratics
    (PAPER.md:534-536): f = x^2 -> Ixx = 128 (sum q)^2, f = y^2 -> Iyy = 128 (sum q)^2,
    f = x y -> Ixy = 64 (sum q)^2, the other components 0; constant -> 0."""
    p = P(width=40, height=36)
    q = oracle.gauss_taps(1.5)
    sq = int(q.sum())
    K = (len(q) - 1) // 2
    yy, xx = np.mgrid[0:36, 0:40]
    ins = _interior(p, K)
    cases = [(xx * xx, (128 * sq * sq, 0, 0)), (yy * yy, (0, 128 * sq * sq, 0)), (xx * yy, (0, 0, 64 * sq * sq)),
             (np.full_like(xx, 999), (0, 0, 0))]
    for f, (exx, eyy, exy) in cases:
        G = oracle.smooth(p, f.astype(np.uint16))
        Ixx, Iyy, Ixy = oracle.hessian(p, G)
        assert np.all(Ixx[ins] == exx) and np.all(Iyy[ins] == eyy) and np.all(Ixy[ins] == exy)


def test_hessian_matches_brute_force_2d():
    """Separable Sobel == direct 5x5 correlation with the outer-product stencils, exactly."""
    rng = np.random.default_rng(7)
    p = P(width=21, height=19)
    G = rng.integers(-10 ** 9, 10 ** 9, size=(19, 21)).astype(np.float64)
    Ixx, Iyy, Ixy = oracle.hessian(p, G)
    for k, (ky, kx) in zip((Ixx, Iyy, Ixy), ((S5, D2), (D2, S5), (D1, D1))):
        st = np.outer(ky, kx)
        ref = np.zeros_like(G)
        for y in range(2, 19 - 2):
            for x in range(2, 21 - 2):
                ref[y, x] = float((st * G[y - 2:y + 3, x - 2:x + 3]).sum())
        assert np.array_equal(k, ref)


# ------------------------------------------------------------------ step 3: eigen
def test_eigen_closed_forms():
    """kappa is the smaller eigenvalue, rho its unit eigenvector."""
    k, dx, dy, deg = oracle.eigen(-2.0, 0.0, -1.0)
    assert (k, abs(dx), dy, deg) == (-2.0, 1.0, 0.0, False)
    k, dx, dy, deg = oracle.eigen(0.0, 1.0, 0.0)
    assert k == -1.0 and not deg
    assert abs(dx * dx + dy * dy - 1) < 1e-15 and dx * dy < 0 and abs(abs(dx) - 2 ** -0.5) < 1e-15
    k, dx, dy, deg = oracle.eigen(5.0, 0.0, 5.0)
    assert deg and k == 5.0


def test_eigen_vs_numpy_eigh():
    """10^4 random integer Hessians vs LAPACK (numpy eigh)."""
    rng = np.random.default_rng(1)
    M = rng.integers(-10 ** 12, 10 ** 12, size=(10000, 3)).astype(np.float64)
    for a, b, c in M:
        k, dx, dy, deg = oracle.eigen(a, b, c)
        w, v = np.linalg.eigh(np.array([[a, b], [b, c]]))
        scale = abs(a) + abs(b) + abs(c)
        assert abs(k - w[0]) <= 1e-12 * scale
        assert abs(abs(dx * v[0, 0] + dy * v[1, 0]) - 1) < 1e-9
        assert abs(math.hypot(dx, dy) - 1) < 1e-15


# ------------------------------------------------------------------ step 4: ridges
def _line_image(W, H, fn):
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    return np.round(100 + fn(xx, yy)).astype(np.uint16)


def test_no_ridges_on_constant_image():
    """kappa = 0 everywhere fails kappa < t <= 0."""
    p = P()
    assert len(oracle.ridges(p, np.full((48, 48), 1234, np.uint16))) == 0


def test_horizontal_line_ridge():
    """A bright horizontal line: ridges are exactly its crest row, direction across the line."""
    p = P()
    img = _line_image(48, 48, lambda x, y: 1000 * np.exp(-(y - 20) ** 2 / (2 * 1.5 ** 2)))
    r = oracle.ridges(p, img)
    assert set(r["y"]) == {20} and sorted(r["x"]) == list(range(3, 48 - 3))
    assert np.all(np.abs(r["dx"]) < 1e-12) and np.all(np.abs(np.abs(r["dy"]) - 1) < 1e-12)


def test_plateau_yields_one_ridge_row():
    """A 2-px-wide plateau (crest between rows 20 and 21): one ridge row, the earlier one
    (reading R6: non-strict after, strict before)."""
    p = P()
    img = _line_image(48, 48, lambda x, y: 1000 * np.exp(-(y - 20.5) ** 2 / (2 * 1.5 ** 2)))
    r = oracle.ridges(p, img)
    assert set(r["y"]) == {20} and len(r) == 48 - 6


def test_vertical_and_diagonal_line_ridges():
    p = P()
    img = _line_image(48, 48, lambda x, y: 1000 * np.exp(-(x - 25) ** 2 / (2 * 1.5 ** 2)))
    r = oracle.ridges(p, img)
    assert set(r["x"]) == {25} and np.all(np.abs(np.abs(r["dx"]) - 1) < 1e-12)
    img = _line_image(48, 48, lambda x, y: 1000 * np.exp(-((x - y) / np.sqrt(2)) ** 2 / (2 * 1.5 ** 2)))
    r = oracle.ridges(p, img)
    on_diag = {(x, x) for x in range(8, 40)}
    got = set(zip(r["x"].tolist(), r["y"].tolist()))
    assert on_diag <= got  # the crest itself
    assert set((r["x"] - r["y"]).tolist()) <= {0, 1}  # 8-neighbour sampling along (1,-1) skips odd offsets
    inner = (r["x"] >= 8) & (r["x"] < 40) & (r["y"] >= 8) & (r["y"] < 40)  # away from the replicate border
    assert np.all(np.abs(np.abs(r["dx"] * r["dy"])[inner] - 0.5) < 1e-12)


def _ring_img(W, H, rings, sigma_p=1.5, pb=2, bg=100):
    sc = synth.scene(W, H, pixel_bytes=pb, max_value=255 if pb == 1 else 4095, background=bg, sigma_p=sigma_p)
    return synth.render(sc, synth.make_rings(rings))


def test_ring_ridges_on_crest_and_radial():
    """Noiseless ring: every ridge lies on the crest (+-1.5 px) and rho is radial to 0.15 rad
    (PAPER.md:308-310 'rho is collinear with the direction to the centre')."""
    p = P(width=96, height=96)
    img = _ring_img(96, 96, [(47.3, 48.6, 25.0, 1500)])
    r = oracle.ridges(p, img)
    d = np.hypot(r["x"] - 47.3, r["y"] - 48.6)
    assert len(r) > 2 * math.pi * 25 * 0.8
    assert np.all(np.abs(d - 25) <= 1.5)
    radial = np.stack([r["x"] - 47.3, r["y"] - 48.6], 1) / d[:, None]
    cosang = np.abs(radial[:, 0] * r["dx"] + radial[:, 1] * r["dy"])
    assert np.all(cosang >= math.cos(0.15))


def test_ridges_translation_equivariant():
    p = P(width=96, height=96)
    a = oracle.ridges(p, _ring_img(96, 96, [(40.0, 44.0, 20.0, 1500)]))
    b = oracle.ridges(p, _ring_img(96, 96, [(47.0, 41.0, 20.0, 1500)]))
    sa = {(x + 7, y - 3, dx, dy) for x, y, dx, dy in zip(a["x"], a["y"], a["dx"], a["dy"])}
    sb = {(x, y, dx, dy) for x, y, dx, dy in zip(b["x"], b["y"], b["dx"], b["dy"])}
    assert sa == sb


# ------------------------------------------------------------------ step 5: votes
def _ridges(rows):
    a = np.zeros(len(rows), dtype=oracle.RIDGE_DTYPE)
    for i, (x, y, dx, dy) in enumerate(rows):
        a[i] = (x, y, dx, dy, -1.0)
    return a


def test_votes_spec_example():
    """ridge (50,50), rho=(1,0), r in [5,6] -> 8 votes at (r,50,50+-r), r=4..7
    (Hough range extended by 1 each side)."""
    p = P(width=128, height=128, r_min=5, r_max=6)
    raw, n = oracle.votes(p, _ridges([(50, 50, 1.0, 0.0)]))
    assert n == 8 and raw.sum() == 8
    for r in range(4, 8):
        lvl = raw[r - 4]
        assert lvl[50, 50 + r] == 1 and lvl[50, 50 - r] == 1


def test_votes_conservation_permutation_duplication():
    """Each vote increments one accumulator by one: sum raw = votes cast in
    frame; an interior ridge casts exactly 2 N_r; order-free; duplicating ridges doubles raw."""
    rng = np.random.default_rng(3)
    p = P(width=200, height=160, r_min=8, r_max=30)
    th = rng.uniform(0, 2 * np.pi, 300)
    rows = [(int(x), int(y), math.cos(t), math.sin(t)) for x, y, t in
            zip(rng.integers(0, 200, 300), rng.integers(0, 160, 300), th)]
    R = _ridges(rows)
    raw, n = oracle.votes(p, R)
    assert raw.sum() == n
    nr = p.r_max - p.r_min + 3
    interior = _ridges([(100, 80, math.cos(t), math.sin(t)) for t in th[:10]])
    assert oracle.votes(p, interior)[1] == 10 * 2 * nr
    raw2, _ = oracle.votes(p, R[rng.permutation(len(R))])
    assert np.array_equal(raw, raw2)
    raw3, n3 = oracle.votes(p, np.concatenate([R, R]))
    assert np.array_equal(raw3, 2 * raw) and n3 == 2 * n
    Rneg = R.copy()
    Rneg["dx"] *= -1
    Rneg["dy"] *= -1
    assert np.array_equal(oracle.votes(p, Rneg)[0], raw)  # eigenvector sign is arbitrary (R8)


def test_votes_gather_brute_force():
    """Gather formulation on a tiny frame: raw[r,y,x] = #{(ridge, s): target == (x,y)}."""
    rng = np.random.default_rng(5)
    p = P(width=24, height=20, r_min=3, r_max=6)
    th = rng.uniform(0, 2 * np.pi, 40)
    R = _ridges([(int(x), int(y), math.cos(t), math.sin(t)) for x, y, t in
                 zip(rng.integers(0, 24, 40), rng.integers(0, 20, 40), th)])
    raw, _ = oracle.votes(p, R)
    for r in range(2, 8):
        for y in range(20):
            for x in range(24):
                cnt = 0
                for rr in R:
                    for s in (1, -1):
                        # round half away from zero, written via Python's Decimal-free floor/ceil
                        ox = math.floor(abs(r * rr["dx"]) + 0.5) * (1 if rr["dx"] >= 0 else -1)
                        oy = math.floor(abs(r * rr["dy"]) + 0.5) * (1 if rr["dy"] >= 0 else -1)
                        cnt += (rr["x"] + s * ox == x) and (rr["y"] + s * oy == y)
                assert raw[r - 2, y, x] == cnt


# ------------------------------------------------------------------ step 7: window sum
def test_window_sum_isolated_count_and_linearity():
    """S of an isolated count c is c * 2^24, i.e. N = c / r (peak weight 1, R11); S is linear."""
    p = P(width=40, height=40, r_min=5, r_max=20)
    r = 16
    raw = np.zeros((oracle.n_levels(p), 40, 40), np.int32)
    raw[r - 4, 17, 23] = 9
    assert oracle.window_sum(p, raw, r, 17, 23) == 9 * 2 ** 24
    rng = np.random.default_rng(2)
    a = rng.integers(0, 50, raw.shape).astype(np.int32)
    b = rng.integers(0, 50, raw.shape).astype(np.int32)
    for (y, x) in ((0, 0), (20, 20), (39, 5)):
        assert oracle.window_sum(p, a + b, r, y, x) == oracle.window_sum(p, a, r, y, x) + oracle.window_sum(p, b, r, y, x)


def test_ideal_ring_scores_two_pi():
    """after smoothing and 1/r normalisation an ideal ring receives ~2 pi votes."""
    lo, hi = GOLDEN["ideal_ring_score"]["accepted_band"]
    for r, sp in ((12, 1.0), (20, 1.5), (35, 1.5), (55, 1.5)):
        W = 2 * r + 40
        p = P(width=W, height=W, r_min=max(3, r - 6), r_max=r + 6, smoothing_sigma=sp)
        img = _ring_img(W, W, [(W // 2, W // 2, float(r), 1500)], sigma_p=sp)
        rings, st = oracle.detect(p, img)
        assert len(rings) == 1
        score = rings[0]["score_fixed"] / (2 ** 24 * rings[0]["r"]) / (2 * math.pi)
        assert lo <= score <= hi


# ------------------------------------------------------------------ step 8: peaks
@pytest.mark.parametrize("sp", [1.0, 1.5])
@pytest.mark.parametrize("r", [8, 12, 20, 33, 47, 60])
def test_exact_recovery_noiseless_ring(r, sp):
    """A noiseless ring with integer centre and radius is recovered exactly as one peak."""
    W = 2 * r + 44
    p = P(width=W, height=W + 6, r_min=6, r_max=64, smoothing_sigma=sp)
    cx, cy = W // 2 - 3, W // 2 + 4
    img = _ring_img(W, W + 6, [(cx, cy, float(r), 1500)], sigma_p=sp)
    rings, _ = oracle.detect(p, img)
    assert [(g["cx"], g["cy"], g["r"]) for g in rings] == [(cx, cy, r)]


def test_two_close_rings_two_peaks():
    """Rings of equal radius 18, centres 25 px apart -> two peaks."""
    p = P(width=110, height=80, r_min=8, r_max=30)
    img = _ring_img(110, 80, [(42, 40, 18.0, 1500), (67, 40, 18.0, 1500)])
    rings, _ = oracle.detect(p, img)
    assert sorted((g["cx"], g["cy"], g["r"]) for g in rings) == [(42, 40, 18), (67, 40, 18)]


def test_peaks_only_inside_search_range():
    """levels r_min-1, r_max+1 are voted but never report peaks."""
    p = P(width=100, height=100, r_min=15, r_max=24)
    img = _ring_img(100, 100, [(30, 30, 14.0, 1500), (68, 66, 25.0, 1500), (70, 25, 19.0, 1500)])
    rings, st = oracle.detect(p, img)
    assert len(rings) >= 1 and all(15 <= g["r"] <= 24 for g in rings)
    assert (70, 25, 19) in [(g["cx"], g["cy"], g["r"]) for g in rings]


def test_plateau_one_peak_lexicographic():
    """Two equal neighbouring maxima: only the lexicographically smaller one is a peak (R14)."""
    p = P(width=16, height=16, r_min=5, r_max=6)
    raw = np.zeros((oracle.n_levels(p), 16, 16), np.int32)
    raw[5 - 4, 8, 8] = 20
    raw[5 - 4, 8, 9] = 20
    pk, hot = oracle.peaks(p, raw)
    assert [(h["r"], h["y"], h["x"]) for h in pk] == [(5, 8, 8)]
    assert len(hot) == 2 and hot[0]["S"] == hot[1]["S"]


def test_peaks_brute_force_small_volumes():
    """Brute-force 3x3x3 maxima of N = S/(2^24 r) over hotspots."""
    rng = np.random.default_rng(11)
    for trial in range(4):
        p = P(width=14, height=12, r_min=4, r_max=7, vote_threshold_raw=3, vote_threshold_norm=0.05)
        raw = rng.integers(0, 12, (oracle.n_levels(p), 12, 14)).astype(np.int32)
        raw[raw < 7] = 0
        pk, hot = oracle.peaks(p, raw)
        Smap = {}
        for h in hot:
            assert h["S"] == oracle.window_sum(p, raw, h["r"], h["y"], h["x"])
            Smap[(int(h["r"]), int(h["y"]), int(h["x"]))] = int(h["S"])
        assert set(Smap) == {(int(r) + 3, int(y), int(x)) for r, y, x in zip(*np.nonzero(raw > 3))}
        expect = []
        for (r, y, x), S in sorted(Smap.items()):
            if not (p.r_min <= r <= p.r_max) or not S > oracle.norm_threshold(p, r):
                continue
            ok = True
            for dr in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        u = (r + dr, y + dy, x + dx)
                        if u == (r, y, x) or not (0 <= u[1] < 12 and 0 <= u[2] < 14):
                            continue
                        Su = Smap.get(u, 0)
                        a, b = S * u[0], Su * r
                        if not (a > b or (a == b and (r, y, x) < u)):
                            ok = False
            if ok:
                expect.append((r, y, x))
        assert [(h["r"], h["y"], h["x"]) for h in pk] == expect


# ------------------------------------------------------------------ step 10: fit
def _pyth(r):
    pts = set()
    for a in range(-r, r + 1):
        b2 = r * r - a * a
        b = int(round(math.sqrt(b2)))
        if b * b == b2:
            pts |= {(a, b), (a, -b)}
    return sorted(pts)


@pytest.mark.parametrize("r", [5, 13, 25])
def test_fit_exact_on_lattice_circle(r):
    """Lattice points exactly on a circle are fitted exactly (Kasa, reading R16)."""
    cx, cy = 40 + 1, 30 - 2  # true centre; the integer peak is off by (1,-2)
    pts = _pyth(r)
    xs = [cx + a for a, b in pts]
    ys = [cy + b for a, b in pts]
    ok, (fx, fy, fr, rms) = oracle.fit(xs, ys, 40, 30)
    assert ok and abs(fx - cx) < 1e-9 and abs(fy - cy) < 1e-9 and abs(fr - r) < 1e-9 and rms < 1e-9


def test_fit_three_points_circumcircle_and_equivariance():
    xs, ys = [0, 10, 3], [0, 1, 9]
    ax, ay, bx, by, cx_, cy_ = 0, 0, 10, 1, 3, 9
    d = 2 * (ax * (by - cy_) + bx * (cy_ - ay) + cx_ * (ay - by))
    ux = ((ax * ax + ay * ay) * (by - cy_) + (bx * bx + by * by) * (cy_ - ay) + (cx_ * cx_ + cy_ * cy_) * (ay - by)) / d
    uy = ((ax * ax + ay * ay) * (cx_ - bx) + (bx * bx + by * by) * (ax - cx_) + (cx_ * cx_ + cy_ * cy_) * (bx - ax)) / d
    ok, (fx, fy, fr, rms) = oracle.fit(xs, ys, 4, 4)
    assert ok and abs(fx - ux) < 1e-9 and abs(fy - uy) < 1e-9 and abs(fr - math.hypot(ux, uy)) < 1e-9
    ok2, (gx, gy, gr, _) = oracle.fit([x + 17 for x in xs], [y - 5 for y in ys], 4 + 17, 4 - 5)
    assert ok2 and abs(gx - fx - 17) < 1e-9 and abs(gy - fy + 5) < 1e-9 and abs(gr - fr) < 1e-9


def test_fit_degenerate_and_residual_bound():
    ok, _ = oracle.fit([0, 1, 2, 3], [0, 1, 2, 3], 0, 0)
    assert not ok  # collinear: singular normal equations
    ok, _ = oracle.fit([0, 1], [0, 5], 0, 0)
    assert not ok  # fewer than 3 inliers
    rng = np.random.default_rng(4)
    th = rng.uniform(0, 2 * np.pi, 80)
    xs = np.round(50 + 20.4 * np.cos(th) + rng.normal(0, 0.4, 80)).astype(int)
    ys = np.round(50 + 20.4 * np.sin(th) + rng.normal(0, 0.4, 80)).astype(int)
    ok, (fx, fy, fr, rms) = oracle.fit(xs, ys, 50, 50)
    int_rms = math.sqrt(np.mean((np.hypot(xs - 50, ys - 50) - 20) ** 2))
    assert ok and rms <= int_rms


# ------------------------------------------------------------------ end to end
def test_end_to_end_exact_recovery_cfg1x():
    """Config "1x" (noiseless cfg1, integer centres): the detected rings are the truth, exactly."""
    p = oracle.params(**synth.preset(11))
    for idx in range(3):
        img, truth = synth.frame(11, 0, idx)
        rings, _ = oracle.detect(p, img)
        got = sorted((g["cx"], g["cy"], g["r"]) for g in rings)
        exp = sorted((int(t["cx"]), int(t["cy"]), int(t["r"])) for t in truth)
        assert got == exp
        for g in rings:
            assert g["fit_ok"] == 1 and abs(g["fr"] - g["r"]) < 0.5


def test_blank_frame_no_rings_and_determinism():
    p = oracle.params(**synth.preset(1))
    rings, st = oracle.detect(p, np.full((128, 128), 20, np.uint8))
    assert len(rings) == 0 and st["ridges"] == 0 and st["votes"] == 0
    img, _ = synth.frame(1, 0, 0)
    a = oracle.detect(p, img)[0]
    b = oracle.detect(p, img)[0]
    assert a.tobytes() == b.tobytes()


def test_ridge_fraction_below_two_percent_cfg3():
    """pixels on the outer rings are < 2 % of the image (cfg3 frame)."""
    p = oracle.params(**synth.preset(3))
    img, _ = synth.frame(3, 0, 0)
    r = oracle.ridges(p, img)
    assert len(r) / img.size < GOLDEN["ring_pixel_fraction"]["max_fraction"]


def test_batch_threads_match_single():
    """Frame-level parallelism does not change results."""
    p = oracle.params(**synth.preset(2))
    frames = synth.batch(2, 0, 0, 3)
    rings, stats = oracle.detect_batch(p, frames, nthreads=3)
    for i in range(3):
        single, st = oracle.detect(p, frames[i])
        assert single.tobytes() == rings[i].tobytes()
        assert st.tobytes() == stats[i].tobytes()


def test_classification_brute_force_annulus():
    """Non-exclusive annulus classification: the inlier count of each
    ring equals a brute-force count of ridges with |distance - r| <= w, w = max(2, ceil(2 sigma(r)))
    with sigma(r) = 0.05 r + 0.25, and a ridge may support several rings."""
    p = oracle.params(**synth.preset(2))
    img, _ = synth.frame(2, 0, 3)
    rings, st, rid, hot = oracle.detect(p, img, want_debug=True)
    assert len(rings) > 5
    used = np.zeros(len(rid), int)
    for g in rings:
        w = max(2, math.ceil(2 * (0.05 * g["r"] + 0.25) - 1e-12))
        d = np.hypot(rid["x"] - g["cx"], rid["y"] - g["cy"])
        m = np.abs(d - g["r"]) <= w + 1e-12
        assert g["inliers"] == int(m.sum())
        used += m
        ok, (fx, fy, fr, rms) = oracle.fit(rid["x"][m], rid["y"][m], g["cx"], g["cy"])
        assert ok == bool(g["fit_ok"]) and abs(fx - g["fx"]) < 1e-9 and abs(fr - g["fr"]) < 1e-9
    assert used.max() >= 1


def test_overlapping_rings_share_ridges():
    """Classification is non-exclusive: pixels at the crossing of two rings support both."""
    p = P(width=110, height=90, r_min=8, r_max=30)
    img = _ring_img(110, 90, [(45, 45, 20.0, 1500), (68, 45, 20.0, 1500)])
    rings, st, rid, hot = oracle.detect(p, img, want_debug=True)
    assert len(rings) == 2
    w = [max(2, math.ceil(2 * (0.05 * g["r"] + 0.25) - 1e-12)) for g in rings]
    both = [(abs(math.hypot(x - rings[0]["cx"], y - rings[0]["cy"]) - rings[0]["r"]) <= w[0]) and
            (abs(math.hypot(x - rings[1]["cx"], y - rings[1]["cy"]) - rings[1]["r"]) <= w[1])
            for x, y in zip(rid["x"], rid["y"])]
    assert sum(both) >= 2
    assert rings["inliers"].sum() == len(rid) + sum(both) - sum(
        1 for x, y in zip(rid["x"], rid["y"])
        if all(abs(math.hypot(x - g["cx"], y - g["cy"]) - g["r"]) > wi for g, wi in zip(rings, w)))
