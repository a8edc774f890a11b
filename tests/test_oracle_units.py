"""Pins of the oracle's integer tables and threshold units (-m "not gpu").

These close the gaps a mutation test of round 1 found: a floor instead of round-half-away in
the smoothing taps or level weights, and a factor 2 in either threshold's units, passed every
earlier pin.  Nothing here re-types the oracle's formulas:

* the tables are compared with golden values (tests/golden/tables.json, SURVEY.md:474) and
  with the reading's definition evaluated in 50-digit decimal arithmetic (Python's
  ``decimal``, an independent exp and rounding);
* the threshold units are fixed by what "counts/px^2" and "counts/px" mean: the gain of a
  brute-force 2D smoothing + Sobel pipeline (written here, in another evaluation order) on
  an image of known curvature (f = x^2) or slope (f = x); then a ridge (edge) whose crest
  curvature (slope) is known in those units must be detected iff it passes the threshold.

tools/mutate_oracle.py applies the four mutations to a copy of oracle.c and checks that
this file fails under each.
"""
import json
import math
import os
from decimal import ROUND_HALF_UP, Decimal, getcontext

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tables.json")))
S5 = np.array([1, 4, 6, 4, 1], dtype=np.int64)
D2 = np.array([1, 0, -2, 0, 1], dtype=np.int64)
D1 = np.array([-1, -2, 0, 2, 1], dtype=np.int64)


def P(**kw):
    base = dict(width=28, height=24, pixel_bytes=2, smoothing_sigma=1.5, curvature_threshold=-10.0, r_min=5,
                r_max=9, vote_threshold_raw=3, vote_threshold_norm=0.5, sig_a=1, sig_b=5, sig_den=20,
                annulus_halfwidth=0, feature=0, edge_threshold=20.0)
    base.update(kw)
    return oracle.params(**base)


def _dec_round(x: Decimal) -> int:
    """Round half away from zero (all values here are positive)."""
    return int(x.quantize(Decimal(1), rounding=ROUND_HALF_UP))


def _dec_taps(sigma: float):
    getcontext().prec = 50
    s = Decimal(repr(sigma))
    K = math.ceil(3 * sigma)
    return [_dec_round(Decimal(1024) * (-Decimal(i * i) / (2 * s * s)).exp()) for i in range(-K, K + 1)]


def _dec_weight(r, d, a=1, b=5, den=20):
    getcontext().prec = 50
    s = Decimal(a * r + b) / Decimal(den)
    return _dec_round(Decimal(4096) * (-Decimal(d * d) / (2 * s * s)).exp())


# ------------------------------------------------------------------ tables
def test_gauss_taps_golden_table():
    """q(sigma_s = 1.5) = [4, 29, 139, 421, 820, 1024, ...], sum 3850 (SURVEY.md:474; R2/R3)."""
    g = GOLD["gauss_taps"]
    q = oracle.gauss_taps(g["sigma_s"])
    assert q.tolist() == g["taps"] and int(q.sum()) == g["sum"]


@pytest.mark.parametrize("sigma", [1.0, 1.2, 1.5, 2.0, 2.5, 3.3, 4.3])
def test_gauss_taps_equal_decimal_definition(sigma):
    """Every tap equals round-half-away(1024 exp(-i^2/(2 sigma^2))) evaluated in 50-digit decimals."""
    assert oracle.gauss_taps(sigma).tolist() == _dec_taps(sigma)


def test_level_weights_golden_table():
    """w_71(0..12) = 4096, 3957, 3566, 2999, 2354, 1724, ... (SURVEY.md:474; R11/R12)."""
    g = GOLD["level_weights"]
    p = P()
    assert oracle.level_halfwidth(p, g["r"]) == g["K"]
    assert [oracle.level_weight(p, g["r"], d) for d in range(g["K"] + 1)] == g["w"]


def test_level_weights_equal_decimal_definition():
    """w_r(d) for every level of the BASELINE configs (r = 4..92) against 50-digit decimals."""
    p = P()
    for r in range(4, 93):
        K = oracle.level_halfwidth(p, r)
        assert K == -(-3 * (r + 5) // 20)
        got = [oracle.level_weight(p, r, d) for d in range(K + 1)]
        assert got == [_dec_weight(r, d) for d in range(K + 1)], r


# ------------------------------------------------------------------ brute-force pipeline
def _brute_smooth(img, q):
    K = (len(q) - 1) // 2
    H, W = img.shape
    pad = np.pad(img.astype(np.int64), K, mode="edge")
    G = np.zeros((H, W), dtype=np.int64)
    for i in range(-K, K + 1):
        for j in range(-K, K + 1):
            G += int(q[i + K]) * int(q[j + K]) * pad[K + i:K + i + H, K + j:K + j + W]
    return G


def _brute_corr(G, ky, kx, y, x):
    st = np.outer(ky, kx)
    return int((st * G[y - 2:y + 3, x - 2:x + 3]).sum())


def _curvature_gain(p):
    """Ixx per count/px^2: the pipeline's response to f = x^2 (f'' = 2 counts/px^2)."""
    W, H = p.width, p.height
    xx = np.mgrid[0:H, 0:W][1]
    G = _brute_smooth((xx - W // 2) ** 2 + 10, oracle.gauss_taps(p.smoothing_sigma))
    return Decimal(_brute_corr(G, S5, D2, H // 2, W // 2)) / 2


def _slope_gain(p):
    """Ix per count/px: the pipeline's response to f = x."""
    W, H = p.width, p.height
    xx = np.mgrid[0:H, 0:W][1]
    G = _brute_smooth(xx + 10, oracle.gauss_taps(p.smoothing_sigma))
    return Decimal(_brute_corr(G, S5, D1, H // 2, W // 2))


@pytest.mark.parametrize("sigma,pb", [(1.5, 2), (1.0, 1), (1.2, 1)])
def test_curvature_threshold_in_counts_per_px2(sigma, pb):
    """The threshold t is in counts/px^2 of the smoothed image (R4/R5):
    in the integer Hessian's units it is t times the pipeline's curvature gain."""
    for t in (-4.0, -10.0, -0.37):
        p = P(smoothing_sigma=sigma, pixel_bytes=pb, curvature_threshold=t)
        # the product is formed in fp64 (one rounding): equal to the exact one within 1 ulp
        assert oracle.curvature_threshold_int(p) == pytest.approx(float(Decimal(repr(t)) * _curvature_gain(p)),
                                                                  rel=2 ** -52)


def _line_ridge(p, profile):
    """A straight ridge along y with profile f(u), u = x - x0, symmetric with a strict minimum
    of the curvature at u = 0: the column x0 is the only directional minimum.  Returns
    (image, x0, crest curvature in counts/px^2 from the brute-force pipeline)."""
    W, H = p.width, p.height
    x0 = W // 2
    u = np.mgrid[0:H, 0:W][1] - x0
    f = profile(u)
    assert f.min() >= 0 and f.max() <= (255 if p.pixel_bytes == 1 else 65535)
    img = f.astype(np.uint8 if p.pixel_bytes == 1 else np.uint16)
    G = _brute_smooth(f, oracle.gauss_taps(p.smoothing_sigma))
    k_int = _brute_corr(G, S5, D2, H // 2, x0)
    assert _brute_corr(G, D2, S5, H // 2, x0) == 0 and _brute_corr(G, D1, D1, H // 2, x0) == 0
    return img, x0, Decimal(k_int) / _curvature_gain(p)


PROFILES = {
    "quartic": lambda u: 1000 - 30 * u * u + u ** 4,             # kappa(u) ~ -60 + 12 u^2 + const
    "quartic_shallow": lambda u: 400 - 22 * u * u + u ** 4,
    "gauss8": lambda u: np.rint(20 + 200 * np.exp(-u * u / 4.5)).astype(np.int64),
}


@pytest.mark.parametrize("sigma,pb,prof", [(1.5, 2, "quartic"), (1.5, 2, "quartic_shallow"), (1.0, 1, "gauss8"),
                                           (1.2, 1, "gauss8")])
def test_ridge_iff_crest_curvature_below_threshold(sigma, pb, prof):
    """A ridge whose crest curvature kappa_c (counts/px^2) is known is detected iff kappa_c < t
    (R4-R6): t just above kappa_c gives exactly the crest column,
    t just below gives nothing."""
    base = dict(smoothing_sigma=sigma, pixel_bytes=pb)
    img, x0, kc = _line_ridge(P(**base), PROFILES[prof])
    assert kc < 0
    eps = abs(kc) * Decimal("0.002")
    above = oracle.ridges(P(**base, curvature_threshold=float(kc + eps)), img)
    H = img.shape[0]
    assert sorted(zip(above["x"].tolist(), above["y"].tolist())) == [(x0, y) for y in range(3, H - 3)]
    assert np.all(np.abs(above["dx"]) == 1.0) and np.all(above["dy"] == 0.0)
    below = oracle.ridges(P(**base, curvature_threshold=float(kc - eps)), img)
    assert len(below) == 0


@pytest.mark.parametrize("sigma", [1.0, 1.5])
def test_edge_threshold_in_counts_per_px(sigma):
    """t_e is in counts/px of the smoothed image (R19): in the squared integer gradient's units
    the threshold is (t_e times the pipeline's slope gain)^2."""
    for te in (10.0, 40.0, 3.25):
        p = P(smoothing_sigma=sigma, feature=1, edge_threshold=te)
        assert oracle.edge_threshold_int2(p) == pytest.approx(float((Decimal(repr(te)) * _slope_gain(p)) ** 2),
                                                              rel=2 ** -50)


def test_edge_iff_crest_slope_above_threshold():
    """An edge whose steepest slope g_c (counts/px) is known is detected iff g_c > t_e
    (R19): f = C + b u - u^3 has its largest |grad| at u = 0 only."""
    p0 = P(feature=1)
    W, H = p0.width, p0.height
    x0 = W // 2
    u = np.mgrid[0:H, 0:W][1] - x0
    f = 8000 + 700 * u - u ** 3
    assert f.min() >= 0 and f.max() <= 65535
    G = _brute_smooth(f, oracle.gauss_taps(1.5))
    gc = Decimal(_brute_corr(G, S5, D1, H // 2, x0)) / _slope_gain(p0)
    assert _brute_corr(G, D1, S5, H // 2, x0) == 0 and gc > 0
    img = f.astype(np.uint16)
    eps = gc * Decimal("0.002")
    below = oracle.ridges(P(feature=1, edge_threshold=float(gc - eps)), img)
    assert sorted(zip(below["x"].tolist(), below["y"].tolist())) == [(x0, y) for y in range(3, H - 3)]
    above = oracle.ridges(P(feature=1, edge_threshold=float(gc + eps)), img)
    assert len(above) == 0


@pytest.mark.parametrize("b", [1.0, -1.0, 3.0, -7.5])
def test_eigen_direction_sign_continuous_from_e_nonnegative(b):
    """R3 puts e = Ixx - Iyy = 0 in the e >= 0 branch: the direction of a matrix with e = 0 is
    the limit of the directions for e -> 0+ (same sign); for b > 0 that is the negation of the
    e -> 0- limit (for b < 0 the two branches agree).
    The sign of rho is part of the ridge record the GPU must reproduce bit for bit."""
    k0, dx0, dy0, _ = oracle.eigen(0.0, b, 0.0)
    kp, dxp, dyp, _ = oracle.eigen(1e-9, b, 0.0)
    km, dxm, dym, _ = oracle.eigen(-1e-9, b, 0.0)
    assert abs(dx0 - dxp) < 1e-6 and abs(dy0 - dyp) < 1e-6
    if b > 0:
        assert abs(dx0 + dxm) < 1e-6 and abs(dy0 + dym) < 1e-6
    assert k0 == -abs(b)
