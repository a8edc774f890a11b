"""Per-config detector parameters (inputs of both the oracle and the CUDA path).

These are workload settings, not method arithmetic: BASELINE.json fixes the frame
shapes and search ranges; the smoothing scale sigma_s = the ring profile sigma
("approximately that of the most visible ring"), and the
thresholds the paper leaves open take the
values of DESIGN.md readings R5, R10, R13.
"""

_BASE = dict(vote_threshold_raw=3, vote_threshold_norm=0.5, sig_a=1, sig_b=5, sig_den=20, annulus_halfwidth=0)

PRESETS = {
    1: dict(smoothing_sigma=1.0, curvature_threshold=-4.0, r_min=5, r_max=30, **_BASE),
    11: dict(smoothing_sigma=1.0, curvature_threshold=-4.0, r_min=5, r_max=30, **_BASE),
    2: dict(smoothing_sigma=1.2, curvature_threshold=-4.0, r_min=6, r_max=45, **_BASE),
    3: dict(smoothing_sigma=1.5, curvature_threshold=-10.0, r_min=8, r_max=70, **_BASE),
    4: dict(smoothing_sigma=1.5, curvature_threshold=-10.0, r_min=8, r_max=90, **_BASE),
    5: dict(smoothing_sigma=1.5, curvature_threshold=-10.0, r_min=8, r_max=70, **_BASE),
}


def preset(cfg: int) -> dict:
    """Full parameter dict (shape + detector settings) of a config."""
    from . import config_shape
    sh = config_shape(cfg)
    d = dict(width=sh["width"], height=sh["height"], pixel_bytes=sh["pixel_bytes"], max_value=sh["max_value"])
    d.update(PRESETS[cfg])
    return d
