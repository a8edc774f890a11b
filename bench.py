#!/usr/bin/env python
"""bench.py — frames/s of the B200 ring detector on BASELINE.json's headline workload.

Step = one pass of the whole hot path (K1 ridges -> K1.5 ray routing -> K2 Hough -> K3
classify/fit -> output) over one batch of B synthetic frames shaped like the paper's workload
(BASELINE.json configs[2]: 1024x688 uint16 (12-bit), 50 rings, overlap / nesting / occlusion;
frames generated with the cfg5 = cfg3 seeds, so frame i is identical for any GPU count).
Frames are resident in HBM before timing; the batch (B * 1.41 MB = 360 MB at B = 256) is
larger than L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl reference]
  python bench.py --config 5 [--gpus N] [--frames 8192] [--parity sample|full|none]

Default (configs[2]): N > 1 is launched by torchrun; each rank processes its own B frames per
step (weak scaling, no data-path collective).  Rank 0 compares every ring of its timed batch
with the CPU oracle ("parity"), which it also times ("cpu_baseline").

--config 5 (BASELINE.json configs[4], the stream sweep): 8192 frames in total, rank k detects
frames [k N/P, (k+1) N/P) in batches of B; after the timed compute the ring lists are gathered
to rank 0 (dist.gather over NCCL); a step = the whole sweep (strong scaling).
Rank 0 reports compute-only and compute+gather frames/s, a sha256 of the gathered records
(identical for every P) and their parity with the oracle.

--impl reference: times the CPU oracle (oracle/, the only reference this paper has) on the
box's host cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = 3                      # BASELINE.json configs[2] (cfg5 frames are cfg3 frames)
WORKLOAD = "cfg3: 1024x688 uint16 (12-bit), 50 rings/frame (30% overlapping pairs, 10% nested, 10% occluded), " \
           "Poisson+read noise; r in [8,70]"
WORKLOAD5 = "cfg5: 8192 frames as cfg3 (seeded per frame index), sharded by frame across the GPUs, ring lists " \
            "gathered to rank 0"
METRIC = "frames/s (0.7 MP, ~50 rings)"
FIT_TOL = 1e-4


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, gpu_index: int, period_ms: int = 50):
        self.gpu, self.period, self.samples, self.proc = gpu_index, period_ms, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        busy = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        reasons = set()
        for s in busy:
            for bit, name in self.REASONS.items():
                if s[2] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in busy), "sm_max_mhz": max(s[1] for s in busy),
                "reasons": sorted(reasons), "samples": len(busy)}


def make_frames(first: int, n: int, out=None):
    import synth
    return synth.batch(CFG, 0, first, n, out=out)


def compare_rings(got: list, exp: list) -> dict:
    """Parity of per-frame ring lists: integer fields bit-exact, fits within FIT_TOL px."""
    bad, worst = [], 0.0
    for i, (g, e) in enumerate(zip(got, exp)):
        ok = g is not None and len(g) == len(e)
        if ok:
            for k in ("cx", "cy", "r", "raw_votes", "score_fixed", "inliers", "fit_ok"):
                ok &= bool(np.array_equal(g[k], e[k]))
            if ok and len(g):
                d = max(float(np.max(np.abs(g[k] - e[k]))) for k in ("fx", "fy", "fr", "rms"))
                worst = max(worst, d)
                ok &= d <= FIT_TOL
        if not ok:
            bad.append(i)
    return {"frames": len(exp), "mismatches": len(bad), "first_mismatch": bad[0] if bad else None,
            "rings": int(sum(len(e) for e in exp)), "max_fit_diff_px": worst, "fit_tol_px": FIT_TOL}


# ------------------------------------------------------------------------ CPU oracle arm
def run_reference(args):
    """The reference arm: the oracle as it stands, on all host cores, a bounded sample per step.
    Workspaces are kept across steps (oracle.Pool), so steps time the arithmetic, not allocation."""
    rank, _, world = _env_rank()
    if rank != 0:
        return 0
    import oracle
    import synth
    per_step = args.ref_frames
    frames = make_frames(0, per_step)
    cores = os.cpu_count() or 1
    pool = oracle.Pool(oracle.params(**synth.preset(CFG)), nthreads=cores)
    for _ in range(max(1, min(args.warmup, 2))):
        pool.detect(frames)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        pool.detect(frames)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = per_step * args.steps / total
    sample = f"frames 0..{per_step - 1} of cfg3 per step, full frames; {cores} threads on {cpu_model()}"
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000 * total / args.steps, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "frames_per_step": per_step, "parallelism": "host threads"},
            "cpu_baseline": {"value": round(value, 3), "unit": "frames/s", "cores": cores, "kind": "oracle",
                             "cpu": cpu_model(), "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------ GPU arm helpers
def _init_dist(args):
    import torch
    import torch.distributed as dist
    rank, local, world = _env_rank()
    if world != args.gpus and world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    return torch, dist, rank, local, world, dev


def _parts(n: int) -> int:
    """Parts rd_detect splits a batch of n frames into (rd_api.cu detect: 3 from 192 frames, 2
    from 128); each part launches K1, K1.5, K2, the redo reset, the 16-bit K2 pass and K3, and
    the call adds k_scan and k_copy."""
    return 3 if n >= 192 else 2 if n >= 128 else 1


def _max_over_ranks(torch, dist, world, dev, v: float) -> float:
    if world > 1:
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        v = float(t.item())
    return v


def run_gpu(args):
    torch, dist, rank, local, world, dev = _init_dist(args)
    import paper_1310_1371_b200 as rd
    import synth

    B = args.batch
    params = synth.preset(CFG)
    fbytes = params["width"] * params["height"] * params["pixel_bytes"]

    # frames of this rank: weak scaling, rank k owns frames [k*B, (k+1)*B)
    frames_h = make_frames(rank * B, B)
    frames_d = torch.from_numpy(frames_h).to(dev)
    det = rd.Detector(params, max_batch=B, device=local)
    out = det.alloc_outputs(B)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        det.detect(frames_d, out, stream)
    det.sync()
    stats = det.stats(B)
    votes_per_step = int(stats["votes"].sum())
    gpu_rings = out.to_numpy()
    # window cells of the hotspots (A7's unit of work): a debug pass over a
    # few frames lists every interior hotspot with its r; cells = sum (2 K_r + 1)^2
    nd = min(B, 8)
    dbg = rd.Detector(dict(params, debug=1), max_batch=nd, device=local)
    dbg.detect(frames_d[:nd])
    dbg.sync()
    win_cells = 0
    hot_per_frame = 0
    for i in range(nd):
        r = dbg.dump_hotspots(i)["r"].astype(np.int64)
        K = (3 * (params["sig_a"] * r + params["sig_b"]) + params["sig_den"] - 1) // params["sig_den"]
        win_cells += int(((2 * K + 1) ** 2).sum())
        hot_per_frame += len(r)
    win_cells_per_frame = win_cells / nd
    hot_per_frame /= nd
    dbg.close()

    # ---------------- timed region: device time, CUDA events on the launching stream
    barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.15)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        det.detect(frames_d, out, stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    ms = e0.elapsed_time(e1)
    # per-kernel durations (the roofline): a separate pass with CUDA events around each kernel
    # on the launching stream (rd_set_timing keeps a batch on one stream: the kernels' own durations)
    det.set_timing(True)
    for _ in range(max(1, min(args.steps, 5))):
        det.detect(frames_d, out, stream)
    kms, ncalls = det.kernel_times()
    det.set_timing(False)
    det.sync()
    clocks = clk.stop()
    ms = _max_over_ranks(torch, dist, world, dev, ms)
    ms_per_step = ms / args.steps
    value = world * B * args.steps / (ms / 1e3)

    # ---------------- end to end through the public API on pinned host buffers
    # Each step is one call with its own H2D of the step's frames and D2H of its rings: the
    # pipelined form keeps two calls in flight (rd_submit_host / rd_wait_host), so a step's
    # copies overlap the previous step's detection; the synchronous rd_detect_host (one call at
    # a time) is reported beside it.
    pinned = torch.from_numpy(frames_h).pin_memory()
    houts = [det.detect_host(pinned), det.detect_host(pinned)]   # host RingBatches allocated once
    e2e_steps = max(1, min(args.steps, args.e2e_steps))

    def e2e_run(pipelined):
        barrier()
        t0 = time.perf_counter()
        if pipelined:
            for i in range(e2e_steps):
                det.submit_host(pinned, houts[i % 2])
                if i >= 1:
                    det.wait_host()
            det.wait_host()
        else:
            for _ in range(e2e_steps):
                det.detect_host(pinned, houts[0])
        dt = time.perf_counter() - t0
        barrier()
        return _max_over_ranks(torch, dist, world, dev, dt)
    e2e_run(True)   # warm-up of the pipelined form
    dt_sync = e2e_run(False)
    dt = e2e_run(True)
    e2e_value = world * B * e2e_steps / dt
    e2e_sync = world * B * e2e_steps / dt_sync
    hout = houts[(e2e_steps - 1) % 2]
    n_rings_rank = int(np.maximum(hout.counts, 0).sum())
    d2h_step = n_rings_rank * 64 + 4 * (2 * B + 1)   # rings found + counts + offsets (compact output)
    host_equal = all(a.tobytes() == b.tobytes() for a, b in zip(hout.to_numpy(), gpu_rings))

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---------------- roofline of the dominant kernel
    names = ["k_ridges", "k_rays", "k_hough", "k_fit"]
    kms_all = [k / ncalls for k in kms]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    px = params["width"] * params["height"]
    Ks = math.ceil(3 * params["smoothing_sigma"])
    # K1 as an fp64/ALU-issue kernel: algorithmic operations per pixel of the exact integer
    # smoothing (2K_s + 1 taps per pass, two passes share the symmetric taps: 2K_s + 1), the
    # Sobel (9 + 9) and the kappa recipe (10); peak = the fp64 pipe, 148 SM x 64/clk x sm_max
    k1_ops_per_px = (2 * Ks + 1) + 9 + 9 + 10
    fp64_peak = 148 * 64 * sm_max * 1e6 / 1e12
    k1_ach = B * px * k1_ops_per_px / (kms_all[0] / 1e3) / 1e12
    # K2 as an ALU-issue-bound kernel: SURVEY.md §8(d)'s count — 11 lane operations per in-frame
    # vote (~10 ops + 1 shared atomic) and 1 per hotspot window cell (one MAC), 3x3x3 NMS compares
    # (26 per hotspot) — against 148 SM x 128 lanes x sm_max
    k2_ops = 11 * votes_per_step + (win_cells_per_frame + 26 * hot_per_frame) * B
    lane_peak = 148 * 128 * sm_max * 1e6 / 1e12
    k2_alu = k2_ops / (kms_all[2] / 1e3) / 1e12
    atom_peak = 11.0 * 148 * sm_max * 1e6 / 1e9   # measured ATOMS/clk/SM (profiles/microbench_r01.log)
    k2_atom = votes_per_step / (kms_all[2] / 1e3) / 1e9
    summ = {}
    sp = os.path.join(ROOT, "profiles", "ncu_summary_r02.json")
    if os.path.exists(sp):
        for d in json.load(open(sp)):
            for n in names:
                if d.get("kernel", "").replace("void ", "").startswith(n) and "dram_bytes_per_frame" in d:
                    summ[n] = d["dram_bytes_per_frame"] * B
    roofs = [
        {"kernel": "k_ridges", "bound": "alu", "achieved": round(k1_ach, 3), "peak": round(fp64_peak, 3),
         "unit": "T op/s", "frac": round(k1_ach / fp64_peak, 4), "traffic": summ.get("k_ridges"),
         "per_unit": f"{k1_ops_per_px} fp64 ops/pixel x {px} pixels x {B} frames per launch",
         "peak_note": "fp64 DFMA issue: 148 SM x 64/clk x sm_max (guide unit counts)"},
        {"kernel": "k_hough", "bound": "alu", "achieved": round(k2_alu, 4), "peak": round(lane_peak, 2),
         "unit": "T lane-op/s", "frac": round(k2_alu / lane_peak, 5), "traffic": summ.get("k_hough"),
         "per_unit": f"11 per in-frame vote ({votes_per_step / B:.0f}/frame) + 1 per window cell "
                     f"({win_cells_per_frame:.0f}/frame) + 26 per hotspot ({hot_per_frame:.0f}/frame) x {B} frames",
         "peak_note": "ALU issue: 148 SM x 128 lanes x sm_max (guide unit counts); SURVEY.md §8(d) op count"},
        {"kernel": "k_hough", "bound": "alu", "achieved": round(k2_atom, 3), "peak": round(atom_peak, 1),
         "unit": "Gvote/s", "frac": round(k2_atom / atom_peak, 5), "traffic": summ.get("k_hough"),
         "peak_note": "shared-memory atomic issue: measured 11.0 ATOMS/clk/SM x 148 SM x sm_max"},
    ]
    dom = 0 if kms_all[0] >= kms_all[2] else 1
    roof = dict(roofs[dom])
    hbm_peak = float(peaks.get("hbm_gbs", 6549.1))
    alg_bytes_frame = fbytes + 64 * (n_rings_rank / B)
    hbm_achieved = alg_bytes_frame * value / world / 1e9

    cpu, parity = None, None
    if not args.no_cpu:
        import oracle
        cores = os.cpu_count() or 1
        n_cpu = min(args.cpu_frames, B)
        pool = oracle.Pool(oracle.params(**params), nthreads=cores)
        pool.detect(frames_h[: min(n_cpu, 2 * cores)])   # workspaces + threads, untimed
        t0 = time.perf_counter()
        exp, est = pool.detect(frames_h[:n_cpu])
        cdt = time.perf_counter() - t0
        pool.close()
        cpu = {"value": round(n_cpu / cdt, 3), "unit": "frames/s", "cores": cores, "kind": "oracle",
               "cpu": cpu_model(),
               "sample": f"the first {n_cpu} frames of this batch (cfg3, full frames), {cdt:.1f} s wall on {cores} "
                         f"threads"}
        parity = compare_rings(gpu_rings[:n_cpu], exp)
        parity["stats_equal"] = bool(all(np.array_equal(stats[k][:n_cpu], est[k][:n_cpu])
                                         for k in ("ridges", "votes", "hotspots", "peaks")))
        parity["host_path_equal_device"] = bool(host_equal)

    line = {"metric": METRIC, "value": round(value, 1), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "frames_per_step_per_gpu": B, "global_batch": B * world,
                       "frame": "1024x688 uint16", "parallelism": f"frame-sharded x{world}",
                       "l2": "inputs larger than L2 (360 MB/step/GPU)"},
            "votes_per_s": round(votes_per_step * world / ms_per_step * 1e3, 1),
            "kernel_ms_per_step": {n: round(k, 4) for n, k in zip(names, kms_all)},
            "roofline": roof,
            "rooflines": roofs,
            "hbm_roofline": {"achieved": round(hbm_achieved, 2), "peak": hbm_peak, "unit": "GB/s",
                             "frac": round(hbm_achieved / hbm_peak, 5),
                             "note": "algorithmic bytes = frame read + 64 B/ring written (SURVEY §8(d))"},
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": {"value": round(e2e_value, 1), "unit": "frames/s", "steps": e2e_steps,
                    "h2d_bytes_per_step": B * fbytes * world, "d2h_bytes_per_step": d2h_step * world,
                    "api": "Detector.submit_host/wait_host -> rd_submit_host/rd_wait_host (pinned host "
                           "buffers, compact ring output, two calls in flight)",
                    "synchronous_value": round(e2e_sync, 1)},
            # K1, K1.5, K2, K2 redo reset, K2 redo pass, K3 per part (a batch of >= 128 frames runs
            # as two halves) + k_scan and k_copy per call
            "gpu_launches": (6 * _parts(B) + 2) * args.steps,
            "clocks": clocks}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------ cfg5 sweep
def run_sweep(args):
    """BASELINE.json configs[4]: 8192 cfg3 frames sharded by frame across P GPUs, ring lists
    gathered to rank 0.  A step = the whole sweep (strong scaling)."""
    torch, dist, rank, local, world, dev = _init_dist(args)
    import paper_1310_1371_b200 as rd
    from paper_1310_1371_b200.distributed import collect, digest, shard, unpack
    import synth

    N, B = args.frames, args.batch
    params = synth.preset(5)
    a, b = shard(N, world, rank)
    n_mine = b - a
    frames_d = torch.empty((n_mine, params["height"], params["width"]), dtype=torch.uint16, device=dev)
    chunk = 512
    for s in range(0, n_mine, chunk):   # generated in pieces (host memory), resident on the device
        m = min(chunk, n_mine - s)
        frames_d[s:s + m].copy_(torch.from_numpy(synth.batch(5, 0, a + s, m)))
    det = rd.Detector(params, max_batch=B, device=local)
    nb = (n_mine + B - 1) // B
    outs = [det.alloc_outputs(min(B, n_mine - k * B)) for k in range(nb)]
    stream = torch.cuda.current_stream(dev)

    def sweep():
        for k in range(nb):
            det.detect(frames_d[k * B:(k + 1) * B], outs[k], stream)

    def gather():
        # this rank's batches, packed, one gather to rank 0 (paper_1310_1371_b200.distributed.collect)
        return collect([(o.rings, o.counts, o.offsets) for o in outs])

    for _ in range(args.warmup):
        sweep()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.15)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(stream)
    for _ in range(args.steps):
        sweep()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ms = _max_over_ranks(torch, dist, world, dev, e0.elapsed_time(e1))
    # compute + gather of one sweep's results (the second gather: the first loads the kernels)
    gather()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    g0 = time.perf_counter()
    res = gather()
    torch.cuda.synchronize(dev)
    gms = _max_over_ranks(torch, dist, world, dev, (time.perf_counter() - g0) * 1e3)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    recs, cnts = res
    sha = digest(recs, cnts)
    lists = unpack(recs, cnts)
    parity = None
    if args.parity != "none":
        import oracle
        cores = os.cpu_count() or 1
        idx = list(range(N)) if args.parity == "full" else sorted(set(np.linspace(0, N - 1, 64).astype(int)))
        pool = oracle.Pool(oracle.params(**params), nthreads=cores)
        exp = []
        for s in range(0, len(idx), 512):
            sel = idx[s:s + 512]
            fr = np.stack([synth.frame(5, 0, i)[0] for i in sel]) if args.parity != "full" else \
                synth.batch(5, 0, sel[0], len(sel))
            exp += pool.detect(fr)[0]
        pool.close()
        parity = compare_rings([lists[i] for i in idx], exp)
        parity["frames_checked"] = "all" if args.parity == "full" else f"{len(idx)} evenly spaced"
    sweep_ms = ms / args.steps
    line = {"metric": METRIC, "value": round(N / (sweep_ms / 1e3), 1), "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sweep_ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD5, "frames_total": N, "frames_per_call": B,
                       "parallelism": f"frame-sharded x{world}, gather to rank 0"},
            "compute_plus_gather": {"value": round(N / ((sweep_ms + gms) / 1e3), 1), "gather_ms": round(gms, 3),
                                    "records": int(recs.shape[0])},
            "gathered_sha256": sha, "parity": parity, "clocks": clocks,
            "gpu_launches": (6 * _parts(B) + 2) * nb * args.steps}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--config", type=int, default=3, choices=[3, 5])
    ap.add_argument("--frames", type=int, default=8192)
    ap.add_argument("--parity", default="sample", choices=["none", "sample", "full"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-frames", type=int, default=256)
    ap.add_argument("--ref-frames", type=int, default=64)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 5:
        if args.steps == 50:
            args.steps = 5   # a step is the whole 8192-frame sweep
        return run_sweep(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
