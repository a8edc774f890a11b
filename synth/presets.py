"""Per-config detector parameters (inputs of both the oracle and the CUDA path).

These are workload settings, not method arithmetic: BASELINE.json fixes the frame
shapes and search ranges; the smoothing scale sigma_s = the ring profile sigma
("approximately that of the most visible ring"), and the
thresholds the paper leaves open take the
values of DESIGN.md readings R5, R10, R13.
"""

_BASE = dict(vote_threshold_raw=3, vote_threshold_norm=0.5, sig_a=1, sig_b=5, sig_den=20, annulus_halfwidth=0,
             feature=0, edge_threshold=0.0)

# Edge variant (NEXT-2, reading R19): |grad| threshold in counts/px of the
# smoothed frame, about a tenth of a ring flank's slope and ~10x the smoothed noise gradient
EDGE_THRESHOLD = {1: 10.0, 11: 10.0, 2: 10.0, 3: 40.0, 4: 40.0, 5: 40.0}

PRESETS = {
    1: dict(smoothing_sigma=1.0, curvature_threshold=-4.0, r_min=5, r_max=30, **_BASE),
    11: dict(smoothing_sigma=1.0, curvature_threshold=-4.0, r_min=5, r_max=30, **_BASE),
    2: dict(smoothing_sigma=1.2, curvature_threshold=-4.0, r_min=6, r_max=45, **_BASE),
    3: dict(smoothing_sigma=1.5, curvature_threshold=-10.0, r_min=8, r_max=70, **_BASE),
    4: dict(smoothing_sigma=1.5, curvature_threshold=-10.0, r_min=8, r_max=90, **_BASE),
    5: dict(smoothing_sigma=1.5, curvature_threshold=-10.0, r_min=8, r_max=70, **_BASE),
}


def edge_preset(cfg: int) -> dict:
    """The config's parameters with directed edges instead of ridges (NEXT-2)."""
    return dict(preset(cfg), feature=1, edge_threshold=EDGE_THRESHOLD[cfg])


def preset(cfg: int) -> dict:
    """Full parameter dict (shape + detector settings) of a config."""
    from . import config_shape
    sh = config_shape(cfg)
    d = dict(width=sh["width"], height=sh["height"], pixel_bytes=sh["pixel_bytes"], max_value=sh["max_value"])
    d.update(PRESETS[cfg])
    return d
