"""GPU parity: the CUDA path (librd.so via the C ABI) against the CPU oracle (-m gpu).

Integer outputs (ridge set incl. the bits of rho, hotspot counts and S, peaks, inlier
counts, stats) must be bit-identical; fitted centre/radius/rms within 1e-4 px
(BASELINE.json north_star).  Inputs: seeded synthetic frames (synth/), the same for
both sides.
"""
import math

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FIT_TOL = 1e-4


@pytest.fixture(scope="module")
def rdmod():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1310_1371_b200 as rd
    return rd


def _det(rdmod, params, max_batch=1, **extra):
    p = dict(params)
    p.update(extra)
    return rdmod.Detector(p, max_batch=max_batch)


def _ridge_set(a, with_kappa=False):
    return {(int(r["x"]), int(r["y"]), float(r["dx"]).hex(), float(r["dy"]).hex()) for r in a}


def _hot_set(a):
    return {(int(h["r"]), int(h["y"]), int(h["x"]), int(h["raw"]), int(h["S"])) for h in a}


def _compare_rings(got, exp):
    assert len(got) == len(exp), (len(got), len(exp))
    for g, e in zip(got, exp):
        for k in ("cx", "cy", "r", "raw_votes", "score_fixed", "inliers", "fit_ok"):
            assert g[k] == e[k], (k, g, e)
        for k in ("fx", "fy", "fr", "rms"):
            assert abs(g[k] - e[k]) <= FIT_TOL, (k, g, e)


def _run(rdmod, params, frames, debug=1, **extra):
    det = _det(rdmod, params, max_batch=len(frames), debug=debug, **extra)
    dev = torch.from_numpy(np.ascontiguousarray(frames)).cuda()
    out = det.detect(dev).to_numpy()
    det.sync()
    return det, out


def _check_frame(rdmod, det, i, params, frame, rings_gpu, full=True):
    p = oracle.params(**params)
    exp_rings, st, rid, hot = oracle.detect(p, frame, want_debug=True)
    _compare_rings(rings_gpu, exp_rings)
    gst = det.stats(i + 1)[i]
    assert (gst["ridges"], gst["votes"], gst["hotspots"], gst["peaks"]) == \
        (st["ridges"], st["votes"], st["hotspots"], st["peaks"])
    if full:
        assert _ridge_set(det.dump_ridges(i)) == _ridge_set(rid)
        assert _hot_set(det.dump_hotspots(i)) == _hot_set(hot)


def _check_batch(det, params, frames, out, n_threads=0):
    """Every frame of a batch against the oracle (rings bit-exact / fits within FIT_TOL, and
    the per-frame counters), computed by the oracle's host thread pool."""
    exp, est = oracle.detect_batch(oracle.params(**params), frames, nthreads=n_threads)
    gst = det.stats(len(frames))
    for i in range(len(frames)):
        assert out[i] is not None, i
        _compare_rings(out[i], exp[i])
        for k in ("ridges", "votes", "hotspots", "peaks"):
            assert gst[k][i] == est[k][i], (i, k)


# ---------------------------------------------------------------- A3 recipe
def test_eigen_recipe_bit_exact(rdmod):
    rng = np.random.default_rng(0)
    M = rng.integers(-10 ** 13, 10 ** 13, size=(12000, 3)).astype(np.float64)
    M[:50] = rng.integers(-3, 4, size=(50, 3))            # small / degenerate-prone
    M[50] = (5.0, 0.0, 5.0)                               # isotropic
    M[51] = (0.0, 1.0, 0.0)
    M[52] = (-2.0, 0.0, -1.0)
    # directions at 30 / 60 degrees, where a component of rho rounds between 0 and 1 (|rho_x| or
    # |rho_y| = 1/2 iff |a - c| = 2|b|/sqrt(3)): the ridge test's neighbour step comes from the
    # squared components there, and inside a 2^-40 band from the exact recipe; magnitudes from
    # 10 (far outside the band after rounding to integers) to 1e13 (inside it)
    for j in range(2000):
        mag = 10.0 ** rng.uniform(1, 13)
        b = float(np.rint(rng.uniform(-1, 1) * mag)) or 1.0
        e = float(np.rint(2.0 * abs(b) / np.sqrt(3.0))) * (1 if j & 1 else -1) + float(rng.integers(-1, 2))
        c = float(np.rint(rng.uniform(-1, 1) * mag))
        M[10000 + j] = (c + e, b, c)
    out, deg = rdmod.eigen(torch.from_numpy(M).cuda())
    out, deg = out.cpu().numpy(), deg.cpu().numpy()
    n_close = 0
    for i, (a, b, c) in enumerate(M):
        k, dx, dy, d = oracle.eigen(a, b, c)
        assert bool(deg[i] & 1) == d
        assert out[i, 0].tobytes() == np.float64(k).tobytes()
        if not d:
            assert out[i, 1].tobytes() == np.float64(dx).tobytes() and out[i, 2].tobytes() == np.float64(dy).tobytes()
            # llround (half away from zero) of the oracle's components
            ox = int(np.sign(dx)) if abs(dx) >= 0.5 else 0
            oy = int(np.sign(dy)) if abs(dy) >= 0.5 else 0
            assert ((deg[i] >> 1) & 3) - 1 == ox and ((deg[i] >> 3) & 3) - 1 == oy, (i, a, b, c, dx, dy, deg[i])
            n_close += min(abs(abs(dx) - 0.5), abs(abs(dy) - 0.5)) < 1e-12
    assert n_close >= 100   # the band's exact path was exercised


# ---------------------------------------------------------------- configs, stage by stage
@pytest.mark.parametrize("cfg", [1, 11])
def test_parity_cfg1(rdmod, cfg):
    params = synth.preset(cfg)
    frames = np.stack([synth.frame(cfg, 0, i)[0] for i in range(4)])
    det, rings = _run(rdmod, params, frames)
    for i in range(4):
        _check_frame(rdmod, det, i, params, frames[i], rings[i])


def test_parity_cfg2_batch16(rdmod):
    params = synth.preset(2)
    frames = synth.batch(2, 0, 0, 16)
    det, rings = _run(rdmod, params, frames)
    for i in range(16):
        _check_frame(rdmod, det, i, params, frames[i], rings[i], full=(i < 4))


def test_parity_cfg3_sample(rdmod):
    params = synth.preset(3)
    frames = synth.batch(3, 0, 0, 4)
    det, rings = _run(rdmod, params, frames)
    for i in range(4):
        _check_frame(rdmod, det, i, params, frames[i], rings[i], full=(i < 2))


def test_parity_cfg4_sample(rdmod):
    params = synth.preset(4)
    frames = synth.batch(4, 0, 0, 2)
    det, rings = _run(rdmod, params, frames, max_entries_per_tile=5120, max_hotspots_per_level=256)
    for i in range(2):
        _check_frame(rdmod, det, i, params, frames[i], rings[i], full=(i < 1))


# ---------------------------------------------------------------- edge cases
def _random_small(seed, W, H, pb):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(0, 5))
    rings = synth.make_rings([(rng.uniform(0, W), rng.uniform(0, H), rng.uniform(4, 25), rng.uniform(200, 1500))
                              for _ in range(n)])
    sc = synth.scene(W, H, pixel_bytes=pb, max_value=255 if pb == 1 else 4095, background=50,
                     sigma_p=rng.uniform(1.0, 2.0), read_sigma=rng.uniform(0, 8), poisson=0)
    return synth.render(sc, rings, noise_key=seed)


@pytest.mark.parametrize("W,H", [(8, 8), (13, 29), (37, 41), (100, 75), (129, 65), (200, 33)])
def test_ragged_and_tiny_frames(rdmod, W, H):
    for pb in (1, 2):
        params = dict(width=W, height=H, pixel_bytes=pb, max_value=255 if pb == 1 else 4095, smoothing_sigma=1.3,
                      curvature_threshold=-4.0 if pb == 1 else -10.0, r_min=3, r_max=min(40, max(W, H)),
                      vote_threshold_raw=2, vote_threshold_norm=0.3, sig_a=1, sig_b=5, sig_den=20,
                      annulus_halfwidth=0)
        frames = np.stack([_random_small(100 * W + H + s + pb, W, H, pb) for s in range(3)])
        det, rings = _run(rdmod, params, frames)
        for i in range(3):
            _check_frame(rdmod, det, i, params, frames[i], rings[i])


def test_blank_and_saturated_frames(rdmod):
    params = synth.preset(2)
    frames = np.stack([np.zeros((480, 640), np.uint8), np.full((480, 640), 255, np.uint8),
                       np.full((480, 640), 17, np.uint8)])
    det, rings = _run(rdmod, params, frames)
    for i in range(3):
        assert len(rings[i]) == 0
        st = det.stats(3)[i]
        assert st["ridges"] == 0 and st["votes"] == 0


def test_rings_at_border_and_fixed_annulus(rdmod):
    params = dict(width=160, height=120, pixel_bytes=2, max_value=4095, smoothing_sigma=1.5,
                  curvature_threshold=-10.0, r_min=6, r_max=50, vote_threshold_raw=3, vote_threshold_norm=0.4,
                  sig_a=1, sig_b=5, sig_den=20, annulus_halfwidth=3)
    sc = synth.scene(160, 120, pixel_bytes=2, max_value=4095, background=100, sigma_p=1.5, read_sigma=4)
    fr = [synth.render(sc, synth.make_rings(spec), noise_key=k) for k, spec in enumerate([
        [(5, 60, 20, 1500), (150, 5, 30, 1500), (80, 118, 15, 1000)],
        [(0, 0, 40, 2000), (159, 119, 25, 2000), (80, 60, 45, 900)],
        [(64, 64, 30, 1500), (64, 64, 12, 1500), (100, 40, 20, 1500, 1.0, 2.5)]])]
    frames = np.stack(fr)
    det, rings = _run(rdmod, params, frames)
    for i in range(3):
        _check_frame(rdmod, det, i, params, frames[i], rings[i])


def test_random_small_frames(rdmod):
    rng = np.random.default_rng(42)
    W, H = 96, 80
    params = dict(width=W, height=H, pixel_bytes=2, max_value=4095, smoothing_sigma=1.5, curvature_threshold=-6.0,
                  r_min=4, r_max=36, vote_threshold_raw=3, vote_threshold_norm=0.35, sig_a=1, sig_b=5, sig_den=20,
                  annulus_halfwidth=0)
    frames = np.stack([_random_small(int(s), W, H, 2) for s in rng.integers(0, 10 ** 6, 24)])
    det, rings = _run(rdmod, params, frames)
    for i in range(len(frames)):
        _check_frame(rdmod, det, i, params, frames[i], rings[i], full=(i < 6))


@pytest.mark.parametrize("seed", range(40))
def test_random_configs(rdmod, seed):
    """A seeded walk over the configuration space rd_create accepts — frame sizes, pixel
    type, smoothing scale, curvature threshold, radius range, both thresholds, the sigma(r)
    rational, fixed annulus widths, ridges or edges — with every stage against the oracle
    (ridge sets incl. the bits of rho, hotspot sets with S, counters, rings).  A config the
    library rejects must be rejected with RD_ERR_PARAM / RD_ERR_DIM / RD_ERR_CONFIG."""
    from paper_1310_1371_b200._rd import RDError, RD_ERR_PARAM, RD_ERR_DIM, RD_ERR_CONFIG
    rng = np.random.default_rng(1000 + seed)
    W, H = int(rng.integers(24, 260)), int(rng.integers(24, 260))
    pb = int(rng.integers(1, 3))
    a, b, den = [(1, 5, 20), (1, 3, 10), (2, 5, 40), (1, 10, 20)][int(rng.integers(0, 4))]
    r_min = int(rng.integers(2, 16))
    r_max = int(min(r_min + rng.integers(1, 100), min(W, H) - 1))
    if r_max <= r_min:
        r_min, r_max = 2, max(3, min(W, H) - 1)
    edge = rng.random() < 0.25
    params = dict(width=W, height=H, pixel_bytes=pb,
                  max_value=255 if pb == 1 else (65535 if rng.random() < 0.25 else 4095),
                  smoothing_sigma=float(rng.uniform(0.7, 4.3)),
                  curvature_threshold=-float(rng.uniform(1, 8) if pb == 1 else rng.uniform(4, 20)),
                  r_min=r_min, r_max=r_max, vote_threshold_raw=int(rng.integers(1, 7)),
                  vote_threshold_norm=float(rng.uniform(0.2, 0.8)), sig_a=a, sig_b=b, sig_den=den,
                  annulus_halfwidth=[0, 0, 1, 3][int(rng.integers(0, 4))],
                  feature=1 if edge else 0, edge_threshold=(10.0 if pb == 1 else 40.0) if edge else 0.0)
    frames = np.stack([_random_small(7919 * seed + k, W, H, pb) for k in range(3)])
    try:
        det, rings = _run(rdmod, params, frames)
    except RDError as e:   # outside what the library takes: rejected with a reason, not run
        assert e.status in (RD_ERR_PARAM, RD_ERR_DIM, RD_ERR_CONFIG), e
        pytest.skip(f"config rejected: {e}")
    for i in range(len(frames)):
        _check_frame(rdmod, det, i, params, frames[i], rings[i])


# ---------------------------------------------------------------- capacities fail loudly
def test_capacity_overflow_reported(rdmod):
    """Every capacity overflow is reported (count -1, flag bit, rd_sync error), and
    rd_query_overflow returns capacities that suffice: a detector recreated with them
    reproduces the oracle's rings (rd.h rd_overflow)."""
    params = synth.preset(2)
    frames = synth.batch(2, 0, 0, 2)
    dev = torch.from_numpy(frames).cuda()
    p = oracle.params(**params)
    exp = [oracle.detect(p, f)[0] for f in frames]
    for extra, bit, key, cfg_key in (
            (dict(max_rings_per_frame=2), 8, "needed_rings_per_frame", "max_rings_per_frame"),
            (dict(max_ridges_per_tile=2), 1, "needed_ridges_per_tile", "max_ridges_per_tile"),
            (dict(max_entries_per_tile=16), 2, "needed_entries_per_tile", "max_entries_per_tile"),
            (dict(max_hotspots_per_level=1), 4, "needed_hotspots_per_level", "max_hotspots_per_level")):
        det = _det(rdmod, params, max_batch=2, **extra)
        out = det.detect(dev)
        with pytest.raises(rdmod.RDError):
            det.sync()
        assert np.all(det.flags(2) & bit) and np.all(out.counts.cpu().numpy() == -1)
        ov = det.overflow()
        assert ov["frames_overflowed"] == 2 and ov["flags"] & bit
        assert ov[key] > extra[cfg_key]
        det2 = _det(rdmod, params, max_batch=2, **{cfg_key: ov[key]})
        got = det2.detect(dev).to_numpy()
        det2.sync()
        assert det2.overflow()["frames_overflowed"] == 0
        for g, e in zip(got, exp):
            _compare_rings(g, e)


def test_sized_for_iterates_to_fitting_capacities(rdmod):
    """Detector.sized_for: from the default capacities, cfg4 (200 dense rings) overflows the ray
    lists; the needed capacities change the Hough tiling, so resizing iterates until nothing
    overflows, and the result equals the oracle."""
    params = synth.preset(4)
    frames = synth.batch(4, 0, 3, 2)
    dev = torch.from_numpy(frames).cuda()
    det = rdmod.Detector.sized_for(params, dev)
    assert det.cfg.max_entries_per_tile > 3072
    out = det.detect(dev).to_numpy()
    det.sync()
    exp, _ = oracle.detect_batch(oracle.params(**params), frames)
    for g, e in zip(out, exp):
        _compare_rings(g, e)


def test_api_state_and_dumps(rdmod):
    """rd.h call order: dumps and stats describe the last rd_detect; after rd_detect_host (whose
    chunks reuse the internal buffers) they return RD_ERR_STATE while rd_query_overflow still
    describes that call; RD_DUMP_MEMBERS equals rd_ring_members back to back."""
    import ctypes as C
    params = synth.preset(2)
    frames = synth.batch(2, 0, 5, 3)
    det = _det(rdmod, params, max_batch=3)
    L = rdmod.lib()
    n = C.c_int64()
    assert L.rd_debug_dump(det._h, 0, 0, None, 0, C.byref(n)) == rdmod._rd.RD_ERR_STATE   # no call yet
    det.detect(torch.from_numpy(frames).cuda())
    det.sync()
    mem = det.ring_members(1)
    flat = det._dump(1, rdmod._rd.RD_DUMP_MEMBERS, np.uint32)
    both = np.concatenate([m[:, 0] | (m[:, 1] << 16) for m in mem]).astype(np.uint32)
    assert np.array_equal(flat, both) and len(flat) > 0
    assert L.rd_debug_dump(det._h, 0, 1, None, 0, C.byref(n)) == rdmod._rd.RD_ERR_STATE   # LEVEL_FPR needs debug
    assert np.all(det.flags(3) == 0)
    det.detect_host(frames)
    assert det.overflow()["frames_overflowed"] == 0
    for bad in (lambda: det.stats(1), lambda: det.flags(1), lambda: det.dump_ridges(0), lambda: det.ring_members(0),
                lambda: det.sync()):
        with pytest.raises(rdmod.RDError):
            bad()


def test_output_capacity_and_offsets(rdmod):
    """Compact output (rd_detect's ring_capacity_total / offsets): frames are back to back;
    a capacity one ring short of the total fails exactly the last frame with OVF_OUTPUT, and
    rd_query_overflow reports the total needed; the host path behaves the same."""
    params = synth.preset(2)
    frames = synth.batch(2, 0, 3, 4)
    det = _det(rdmod, params, max_batch=4)
    full = det.detect(torch.from_numpy(frames).cuda())
    det.sync()
    counts, offsets = full.counts.cpu().numpy(), full.offsets.cpu().numpy()
    total = int(offsets[-1])
    assert offsets[0] == 0 and np.array_equal(np.diff(offsets), counts) and total == counts.sum() > 0
    assert det.overflow()["needed_rings_total"] == total
    short = det.detect(torch.from_numpy(frames).cuda(), det.alloc_outputs(4, capacity=total - 1))
    assert det.sync(raise_on_overflow=False) == rdmod._rd.RD_ERR_CAPACITY
    c2 = short.counts.cpu().numpy()
    assert np.array_equal(c2[:3], counts[:3]) and c2[3] == -1
    assert det.flags(4)[3] & 32 and det.overflow()["needed_rings_total"] == total
    a, b = full.to_numpy(), short.to_numpy()
    for i in range(3):
        assert a[i].tobytes() == b[i].tobytes()
    hb = det.detect_host(frames, capacity=total - 1)
    assert np.array_equal(hb.counts[:3], counts[:3]) and hb.counts[3] == -1
    ov = det.overflow()
    assert ov["needed_rings_total"] == total and ov["frames_overflowed"] == 1 and ov["flags"] & 32
    hb = det.detect_host(frames, capacity=total)
    assert np.array_equal(hb.counts, counts) and np.array_equal(hb.offsets, offsets)


def test_invalid_config_rejected(rdmod):
    base = synth.preset(2)
    for bad in (dict(smoothing_sigma=0.0), dict(curvature_threshold=1.0), dict(r_min=1), dict(r_max=3, r_min=5),
                dict(vote_threshold_raw=0), dict(vote_threshold_norm=-1.0), dict(width=4)):
        with pytest.raises(rdmod.RDError):
            _det(rdmod, base, **bad)


# ---------------------------------------------------------------- full size, bench launch configuration
def test_full_batch_cfg3_bench_config(rdmod):
    """cfg3 at BASELINE size (256 frames, the bench step, same launch configuration): every
    frame vs the oracle; canonical order, range and determinism."""
    params = synth.preset(3)
    frames = synth.batch(3, 0, 0, 256)
    det = _det(rdmod, params, max_batch=256)
    dev = torch.from_numpy(frames).cuda()
    out = det.detect(dev).to_numpy()
    det.sync()
    out2 = det.detect(dev).to_numpy()
    det.sync()
    assert all(a.tobytes() == b.tobytes() for a, b in zip(out, out2))  # deterministic
    _check_batch(det, params, frames, out)   # all 256 frames of the bench step
    for g in out:
        assert g is not None and len(g) > 20
        key = list(zip(g["r"], g["cy"], g["cx"]))
        assert key == sorted(key) and len(set(key)) == len(key)
        assert np.all((g["r"] >= params["r_min"]) & (g["r"] <= params["r_max"]))
        assert np.all(g["score_fixed"] > 0.5 * 2 * math.pi * 2 ** 24 * g["r"])
    st = det.stats(256)
    assert np.all(st["votes"] > 10 ** 6)


def test_detect_host_matches_device(rdmod):
    params = synth.preset(3)
    frames = synth.batch(3, 0, 300, 70)
    det = _det(rdmod, params, max_batch=70)
    dev_out = det.detect(torch.from_numpy(frames).cuda()).to_numpy()
    det.sync()
    pinned = torch.from_numpy(frames).pin_memory()
    hb = det.detect_host(pinned)
    host_out = hb.to_numpy()
    for i in range(70):
        assert hb.counts[i] == len(dev_out[i])
        assert host_out[i].tobytes() == dev_out[i].tobytes()
    # compact output: the rings of all frames back to back, nothing else read back
    assert hb.offsets[0] == 0 and np.array_equal(np.diff(hb.offsets), hb.counts)


@pytest.mark.parametrize("force_redo", [False, True])
def test_detect_host_many_chunks_two_slots(rdmod, force_redo, monkeypatch):
    """rd_detect_host with n_frames far above max_batch: ramped chunks alternate between two
    streams on disjoint halves of the internal buffers (frame views with their own K2 work
    counters and redo lists); every frame equals the device path, also when every frame
    takes the 16-bit redo pass."""
    if force_redo:
        monkeypatch.setenv("RD_K2_FORCE_REDO", "1")
    params = synth.preset(2)
    frames = synth.batch(2, 0, 40, 37)
    det = _det(rdmod, params, max_batch=8)
    ref = []
    for i in range(0, 37, 8):
        ref += det.detect(torch.from_numpy(frames[i:i + 8]).cuda()).to_numpy()
        det.sync()
    host_out = det.detect_host(torch.from_numpy(frames).pin_memory()).to_numpy()
    for i in range(37):
        assert len(host_out[i]) == len(ref[i]) > 0
        assert host_out[i].tobytes() == ref[i].tobytes()


@pytest.mark.parametrize("force_redo", [False, True])
def test_submit_host_pipelined_equals_device_path(rdmod, force_redo, monkeypatch):
    """rd_submit_host / rd_wait_host: five calls of different frames and sizes with two in
    flight (the copies of a call overlap the previous call's detection, its chunks continue
    the stage and slot rotation) give every frame the device path's rings, the oldest call
    completing first; also when every frame takes the 16-bit redo pass."""
    if force_redo:
        monkeypatch.setenv("RD_K2_FORCE_REDO", "1")
    params = synth.preset(2)
    sizes = [19, 7, 1, 23, 12]
    batches = [synth.batch(2, 100 + i, 100 + i + m, m) for i, m in enumerate(sizes)]
    det = _det(rdmod, params, max_batch=8)
    ref = []
    for b in batches:
        r = []
        for i in range(0, len(b), 8):
            r += det.detect(torch.from_numpy(b[i:i + 8]).cuda()).to_numpy()
            det.sync()
        ref.append(r)
    pinned = [torch.from_numpy(b).pin_memory() for b in batches]
    got, outs = [], []
    for i, p in enumerate(pinned):
        outs.append(det.submit_host(p))
        if i >= 1:
            got.append(det.wait_host())
    got.append(det.wait_host())
    assert [g is o for g, o in zip(got, outs)] == [True] * len(sizes)
    for b, (g, r) in enumerate(zip(got, ref)):
        g = g.to_numpy()
        assert len(g) == sizes[b]
        for i in range(sizes[b]):
            assert g[i].tobytes() == r[i].tobytes(), (b, i)
    assert det.overflow()["frames_overflowed"] == 0


def test_submit_host_state_rules(rdmod):
    """rd.h: at most RD_HOST_DEPTH calls in flight; waiting with none in flight, and
    rd_detect_host / rd_detect / queries with calls in flight are RD_ERR_STATE; after the
    waits rd_detect and rd_query_overflow work and describe the right call."""
    L, R = rdmod.lib(), rdmod._rd
    params = synth.preset(2)
    frames = synth.batch(2, 0, 6, 6)
    det = _det(rdmod, params, max_batch=6)
    assert L.rd_wait_host(det._h) == R.RD_ERR_STATE
    a = det.submit_host(frames)
    b = det.submit_host(frames[:3], capacity=1)   # too small: RD_ERR_CAPACITY at its wait
    with pytest.raises(rdmod.RDError):
        det.submit_host(frames)
    for bad in (lambda: det.detect_host(frames), lambda: det.detect(torch.from_numpy(frames).cuda()),
                lambda: det.overflow(), lambda: det.sync()):
        with pytest.raises(rdmod.RDError) as e:
            bad()
        assert e.value.status == R.RD_ERR_STATE
    assert det.wait_host() is a and np.all(a.counts >= 0)
    with pytest.raises(rdmod.RDError):   # b still in flight
        det.overflow()
    assert det.wait_host() is b
    assert b.counts[0] == -1 or b.counts[0] <= 1
    ov = det.overflow()
    assert ov["frames_overflowed"] >= 1 and ov["needed_rings_total"] == a.offsets[3]
    dev = det.detect(torch.from_numpy(frames).cuda())
    det.sync()
    assert np.array_equal(dev.counts.cpu().numpy(), a.counts)
    assert L.rd_wait_host(det._h) == R.RD_ERR_STATE


@pytest.mark.parametrize("cfg", [2, 3])
def test_ring_members_match_annulus_definition(rdmod, cfg):
    """rd_ring_members (A9): every ring's members are exactly the oracle's ridge pixels in
    its annulus (r-w)_+^2 <= d^2 <= (r+w)^2, as many as the
    ring's inliers, in ridge-bin order (bin row, bin column, row-major inside a bin)."""
    params = synth.preset(cfg)
    frames = synth.batch(cfg, 0, 7, 2)
    det = _det(rdmod, params, max_batch=2)
    out = det.detect(torch.from_numpy(frames).cuda()).to_numpy()
    det.sync()
    p = oracle.params(**params)
    for i in range(2):
        R = oracle.ridges(p, frames[i])
        rx, ry = R["x"].astype(np.int64), R["y"].astype(np.int64)
        mem = det.ring_members(i)
        assert len(mem) == len(out[i]) > 0
        for ring, m in zip(out[i], mem):
            r = int(ring["r"])
            w = oracle.annulus_halfwidth(p, r)
            lo, hi = max(r - w, 0), r + w
            d2 = (rx - int(ring["cx"])) ** 2 + (ry - int(ring["cy"])) ** 2
            sel = (d2 >= lo * lo) & (d2 <= hi * hi)
            assert len(m) == int(ring["inliers"]) == int(sel.sum())
            assert {(int(a), int(b)) for a, b in zip(rx[sel], ry[sel])} == {(int(a), int(b)) for a, b in m}
            key = [(int(y) // 32, int(x) // 32, int(y), int(x)) for x, y in m]
            assert key == sorted(key)


@pytest.mark.parametrize("n", [193, 200])
def test_batch_parts_do_not_change_results(rdmod, n, monkeypatch):
    """rd_detect runs a large batch as two or three parts on internal streams (frame views of
    the internal buffers; three from 192 frames).  Ragged part boundaries and every part count
    give the same ring lists, counts and per-frame counters as one part."""
    params = synth.preset(2)
    frames = torch.from_numpy(synth.batch(2, 0, 0, n)).cuda()
    det = _det(rdmod, params, max_batch=n)
    monkeypatch.setenv("RD_SPLIT", "1")
    ref = det.detect(frames).to_numpy()
    det.sync()
    ref_st = det.stats(n)
    for split in ("2", "3", "4", None):
        if split is None:
            monkeypatch.delenv("RD_SPLIT")
        else:
            monkeypatch.setenv("RD_SPLIT", split)
        out = det.detect(frames).to_numpy()
        det.sync()
        assert [a.tobytes() for a in out] == [a.tobytes() for a in ref], split
        st = det.stats(n)
        for k in ("ridges", "votes", "hotspots", "peaks"):
            assert np.array_equal(st[k], ref_st[k]), (split, k)


@pytest.mark.parametrize("env", [("RD_K2_SQUARE", "1"), ("RD_K2_TILE", "86,77"), ("RD_K2_TILE", "200,60"),
                                 ("RD_K2_RR16", "0")])
def test_rings_independent_of_hough_tiling(rdmod, env, monkeypatch):
    """The Hough tiling (square, rectangular, thin) changes how K1.5 routes rays and K2
    sweeps tiles, never the result: every frame's ring list is byte-identical to the default
    tiling's.  So does K2's ray storage: 2-byte level intervals all resident (the default
    below 255 levels) or 4-byte intervals with the first rays resident (RD_K2_RR16=0)."""
    params = synth.preset(3)
    frames = torch.from_numpy(synth.batch(3, 0, 60, 6)).cuda()
    det = _det(rdmod, params, max_batch=6)
    ref = det.detect(frames).to_numpy()
    det.sync()
    monkeypatch.setenv(*env)
    det2 = _det(rdmod, params, max_batch=6)
    out = det2.detect(frames).to_numpy()
    det2.sync()
    for a, b in zip(ref, out):
        assert len(a) > 20 and a.tobytes() == b.tobytes()


def test_full_batch_cfg4_dense(rdmod):
    """cfg4 at BASELINE size (512 frames of 1024x1024, 200 rings): every frame vs the oracle
    (no capacity overflow with the dense-config capacities)."""
    params = dict(synth.preset(4), max_entries_per_tile=5120, max_hotspots_per_level=256)
    frames = synth.batch(4, 0, 0, 512)
    det = _det(rdmod, params, max_batch=512)
    out = det.detect(torch.from_numpy(frames).cuda()).to_numpy()
    det.sync()
    assert all(g is not None and len(g) > 100 for g in out)
    _check_batch(det, params, frames, out)


def test_cfg5_high_frame_indices(rdmod):
    """cfg5 (8192 frames = cfg3 seeds, sharded by frame): the last 256 frames as one rank's
    batch; frame content is independent of the sharding (synth keys by frame index)."""
    params = synth.preset(5)
    frames = synth.batch(5, 0, 8192 - 256, 256)
    assert np.array_equal(frames[-1], synth.frame(3, 0, 8191)[0])
    det = _det(rdmod, params, max_batch=256)
    out = det.detect(torch.from_numpy(frames).cuda()).to_numpy()
    det.sync()
    _check_batch(det, params, frames, out)


def test_detect_host_pitched_frames(rdmod):
    """rd_detect_host with a row pitch wider than the frame (non-contiguous rows)."""
    params = synth.preset(2)
    frames = synth.batch(2, 0, 20, 5)
    padded = np.zeros((5, 480, 704), np.uint8)
    padded[:, :, :640] = frames
    det = _det(rdmod, params, max_batch=3)
    out = det.detect_host(padded[:, :, :640]).to_numpy()
    p = oracle.params(**params)
    for i in range(5):
        _compare_rings(out[i], oracle.detect(p, frames[i])[0])


# ---------------------------------------------------------------- K2 counter width
@pytest.mark.parametrize("knob", [("RD_K2_FORCE_REDO", "1"), ("RD_K2_U8_LIMIT", "170"), ("RD_K2_CB", "2")])
def test_k2_counter_width_paths_bit_exact(rdmod, knob, monkeypatch):
    """Byte counters are exact below 255; a frame whose counter reaches the limit is
    recomputed with 16-bit counters.  Forcing every frame through the redo pass, lowering
    the limit to 170 so that only some frames take it (the oracle's raw maxima of these
    six frames are 187, 184, 157, 169, 166, 171: frames 0, 1, 5 are redone), or running
    16-bit counters only must all give the oracle's results bit for bit."""
    monkeypatch.setenv(*knob)
    params = synth.preset(3)
    frames = synth.batch(3, 0, 0, 6)
    det, rings = _run(rdmod, params, frames)
    for i in range(6):
        _check_frame(rdmod, det, i, params, frames[i], rings[i], full=(i < 2))


# ---------------------------------------------------------------- NEXT-2: directed edges
@pytest.mark.parametrize("cfg,n,full", [(1, 4, 4), (2, 4, 2), (3, 2, 1)])
def test_edge_variant_parity(rdmod, cfg, n, full):
    """The directed-edge variant (reading R19: 5x5 first-order Sobel,
    |grad|^2 a local maximum along the gradient) against the oracle: edge sets with the bits
    of rho, hotspots, peaks and stats bit-exact, fits within 1e-4 px."""
    params = synth.edge_preset(cfg)
    frames = np.stack([synth.frame(cfg, 0, i)[0] for i in range(n)]) if cfg == 1 else synth.batch(cfg, 0, 0, n)
    det, rings = _run(rdmod, params, frames, max_entries_per_tile=4096)
    for i in range(n):
        _check_frame(rdmod, det, i, params, frames[i], rings[i], full=(i < full))


def test_edge_config_validated(rdmod):
    """feature must be 0 or 1; edges need a positive, finite edge_threshold."""
    base = synth.preset(3)
    for bad in (dict(feature=2), dict(feature=1, edge_threshold=0.0), dict(feature=1, edge_threshold=-3.0)):
        with pytest.raises(rdmod.RDError):
            _det(rdmod, dict(base, **bad))
    _det(rdmod, dict(base, feature=1, edge_threshold=5.0)).close()


# ---------------------------------------------------------------- NEXT-3: robustness corpus
def test_robustness_corpus_gpu_equals_oracle(rdmod):
    """The GPU rings on the robustness corpus (PAPER.md:611-627 shape) are the oracle's, and
    their detection rate is what the method reaches there (> 90 %)."""
    from synth import robust
    frames, truth = robust.corpus(2026, 32)
    det, rings = _run(rdmod, robust.PARAMS, frames, debug=0)
    exp, _ = oracle.detect_batch(oracle.params(**robust.PARAMS), frames)
    for g, e in zip(rings, exp):
        _compare_rings(g, e)
    rates, _ = robust.score(truth, rings)
    assert rates["detection_rate"] > 0.9 and rates["false_rate"] < 0.05


# ---------------------------------------------------------------- NEXT-4: streaming ingest
def test_stream_detector_matches_batch(rdmod):
    """Frames pushed one at a time (a 500 Hz producer thread) through StreamDetector give the
    batch detector's rings, every frame reported once, in order."""
    import threading
    import time
    from paper_1310_1371_b200.stream import StreamDetector
    params = synth.preset(2)
    frames = synth.batch(2, 0, 0, 16)
    det, ref = _run(rdmod, params, frames, debug=0)
    sd = StreamDetector(params, slots=8, max_batch=4)
    seen = []

    def on_result(i, rings, dt):
        seen.append(i)
        _compare_rings(rings, ref[i % 16])

    cons = threading.Thread(target=sd.run, kwargs=dict(on_result=on_result))
    cons.start()
    for i in range(40):
        sd.push(frames[i % 16])
        time.sleep(0.002)
    sd.close()
    cons.join()
    assert seen == list(range(40))


# ---------------------------------------------------------------- T3: level fingerprints
@pytest.mark.parametrize("cfg,idx", [(2, 0), (3, 5)])
def test_level_fingerprints_match_oracle_accumulator(rdmod, cfg, idx):
    """RD_DUMP_LEVEL_FPR: per level r, sum raw, sum raw^2 and sum raw*(yW+x)
    over every voxel of the frame's raw accumulator equal the oracle's full (N_r x H x W) array
    built from its own ridges (votes populate the levels)."""
    params = synth.preset(cfg)
    frames = synth.batch(cfg, 0, idx, 2)
    det, _ = _run(rdmod, params, frames)
    p = oracle.params(**params)
    W = params["width"]
    for i in range(2):
        raw, nv = oracle.votes(p, oracle.ridges(p, frames[i]))
        raw = raw.astype(np.int64).reshape(raw.shape[0], -1)
        pos = np.arange(raw.shape[1], dtype=np.uint64)
        fpr = det.dump_level_fpr(i)
        assert len(fpr) == raw.shape[0] and np.array_equal(fpr["r"], np.arange(p.r_min - 1, p.r_max + 2))
        assert np.array_equal(fpr["votes"], raw.sum(axis=1)) and int(fpr["votes"].sum()) == nv
        assert np.array_equal(fpr["sq"], (raw * raw).sum(axis=1))
        got_pos = fpr["pos"].astype(np.uint64)
        exp_pos = np.array([int((raw[l].astype(np.uint64) * pos).sum(dtype=np.uint64)) for l in range(raw.shape[0])],
                           dtype=np.uint64)
        assert np.array_equal(got_pos, exp_pos)
        assert W > 0


# ---------------------------------------------------------------- parameter extremes
@pytest.mark.parametrize("r_min,r_max", [(60, 100), (80, 150)])
def test_large_radius_wide_windows(rdmod, r_min, r_max):
    """r_max >= 95 gives K_r = ceil(3 sigma(r)) >= 16: window sums of 2K + 1 > 32 rows, so
    the 16-bit K2 pass sums several rows per lane (sigma(r) grows with r)."""
    W = H = 384
    params = dict(width=W, height=H, pixel_bytes=2, max_value=4095, smoothing_sigma=1.5,
                  curvature_threshold=-10.0, r_min=r_min, r_max=r_max, vote_threshold_raw=3,
                  vote_threshold_norm=0.5, sig_a=1, sig_b=5, sig_den=20, annulus_halfwidth=0)
    sc = synth.scene(W, H, pixel_bytes=2, max_value=4095, background=100, sigma_p=1.5, read_sigma=8, poisson=1)
    rng = np.random.default_rng(r_max)
    fr = []
    for k in range(3):
        rings = [(rng.uniform(r_max * 0.6, W - r_max * 0.6), rng.uniform(r_max * 0.6, H - r_max * 0.6),
                  rng.uniform(r_min + 2, r_max - 2), rng.uniform(800, 3000)) for _ in range(3)]
        fr.append(synth.render(sc, synth.make_rings(rings), noise_key=1000 + k))
    frames = np.stack(fr)
    det, rings = _run(rdmod, params, frames)
    Kmax = -(-3 * (r_max + 1 + 5) // 20)
    assert Kmax >= 16
    for i in range(3):
        assert len(rings[i]) >= 1
        _check_frame(rdmod, det, i, params, frames[i], rings[i])


def test_largest_smoothing_scale(rdmod):
    """sigma_s = 4.3 (K_s = 13, the largest the K1 halo takes): parity on small frames."""
    W, H = 200, 150
    params = dict(width=W, height=H, pixel_bytes=2, max_value=4095, smoothing_sigma=4.3,
                  curvature_threshold=-0.5, r_min=8, r_max=50, vote_threshold_raw=3,
                  vote_threshold_norm=0.3, sig_a=1, sig_b=5, sig_den=20, annulus_halfwidth=0)
    sc = synth.scene(W, H, pixel_bytes=2, max_value=4095, background=100, sigma_p=4.0, read_sigma=4)
    frames = np.stack([synth.render(sc, synth.make_rings([(70, 70, 35, 2500), (140, 80, 25, 2500)]), noise_key=k)
                       for k in range(2)])
    det, rings = _run(rdmod, params, frames)
    for i in range(2):
        _check_frame(rdmod, det, i, params, frames[i], rings[i])
