#!/usr/bin/env python
"""bench.py — frames/s of the B200 ring detector on BASELINE.json's headline workload.

Step = one pass of the whole hot path (K1 ridges -> K2 Hough -> K3 classify/fit) over one
batch of B synthetic frames shaped like the paper's workload (BASELINE.json configs[2]:
1024x688 uint16 (12-bit), 50 rings, overlap / nesting / occlusion; frames generated as
cfg5 = cfg3 seeds, so frame i is identical for any GPU count).  Frames are resident in HBM
before timing; the batch (B * 1.41 MB = 360 MB at B = 256) is larger than L2, so no
flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl reference]

N > 1: launched by torchrun; each rank processes its own B frames per step (weak
scaling, no data-path collective); after the timed region the ring lists are gathered
to rank 0 over NCCL (the paper's producer/consumer result collection)
and checked for P-invariance of frame content.

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
METRIC = "frames/s (0.7 MP, ~50 rings)"


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


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


def make_frames(first: int, n: int):
    import synth
    return synth.batch(CFG, 0, first, n)


# ------------------------------------------------------------------------ CPU oracle arm
def cpu_oracle_rate(n_frames: int, first: int = 0, frames=None, streamed: bool = False):
    """Time the oracle (as it stands) on all host cores over a bounded sample.  streamed=True
    times the paper's own streamed CPU method (oracle/streamed.c, NEXT-1) instead."""
    import oracle
    import synth
    p = oracle.params(**synth.preset(CFG))
    if frames is None:
        frames = make_frames(first, n_frames)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.detect_batch(p, frames, nthreads=cores, streamed=streamed)
    dt = time.perf_counter() - t0
    return n_frames / dt, cores, dt


def run_reference(args):
    rank, _, world = _env_rank()
    if rank != 0:
        return 0
    import synth  # noqa: F401
    per_step = args.ref_frames
    frames = make_frames(0, per_step)
    cpu_oracle_rate(min(per_step, 4), frames=frames[: min(per_step, 4)])  # warm (page faults, threads)
    for _ in range(max(0, min(args.warmup, 1))):
        pass
    times = []
    cores = os.cpu_count() or 1
    for _ in range(args.steps):
        _, cores, dt = cpu_oracle_rate(per_step, frames=frames)
        times.append(dt)
    total = sum(times)
    value = per_step * args.steps / total
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000 * total / args.steps, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "frames_per_step": per_step, "parallelism": "host threads"},
            "cpu_baseline": {"value": round(value, 3), "unit": "frames/s", "cores": cores, "kind": "oracle",
                             "sample": f"frames 0..{per_step - 1} of cfg3 per step, full frames"},
            "e2e": {"value": round(value, 3), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1310_1371_b200 as rd
    import synth

    rank, local, world = _env_rank()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    B = args.batch
    params = synth.preset(CFG)
    fbytes = params["width"] * params["height"] * params["pixel_bytes"]

    # frames of this rank: weak scaling, rank k owns frames [k*B, (k+1)*B)
    frames_h = make_frames(rank * B, B)
    frames_d = torch.from_numpy(frames_h).to(dev)
    det = rd.Detector(params, max_batch=B, device=local)
    rings, counts = det.alloc_outputs(B)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        det.detect(frames_d, rings, counts, stream)
    det.sync()
    stats = det.stats(B)
    votes_per_step = int(stats["votes"].sum())
    # window cells of the hotspots (A7's unit of work): a debug pass over a
    # few frames lists every interior hotspot with its r; cells = sum (2 K_r + 1)^2
    nd = min(B, 8)
    dbg = rd.Detector(dict(params, debug=1), max_batch=nd, device=local)
    dbg.detect(frames_d[:nd])
    dbg.sync()
    win_cells = 0
    for i in range(nd):
        r = dbg.dump_hotspots(i)["r"].astype(np.int64)
        K = (3 * (params["sig_a"] * r + params["sig_b"]) + params["sig_den"] - 1) // params["sig_den"]
        win_cells += int(((2 * K + 1) ** 2).sum())
    win_cells_per_frame = win_cells / nd
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
        det.detect(frames_d, rings, counts, stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    ms = e0.elapsed_time(e1)
    # per-kernel durations (the roofline): a separate pass with CUDA events around each kernel
    # on the launching stream; timing keeps a batch on one stream (no two-half overlap), so
    # these are the kernels' own durations
    det.set_timing(True)
    for _ in range(max(1, min(args.steps, 5))):
        det.detect(frames_d, rings, counts, stream)
    kms, ncalls = det.kernel_times()
    det.set_timing(False)
    det.sync()
    clocks = clk.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * B * args.steps / (ms / 1e3)

    # ---------------- end to end through the public API on pinned host buffers
    pinned = torch.from_numpy(frames_h).pin_memory()
    h_rings = torch.empty((B, det.ring_cap, rd.RING_DTYPE.itemsize), dtype=torch.uint8).pin_memory()
    h_counts = torch.empty((B,), dtype=torch.int32).pin_memory()
    for _ in range(max(1, min(args.warmup, 2))):
        det.detect_host(pinned, h_rings, h_counts)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        det.detect_host(pinned, h_rings, h_counts)
    dt = time.perf_counter() - t0
    barrier()
    if world > 1:
        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    e2e_value = world * B * e2e_steps / dt

    # ---------------- gather ring lists to rank 0 over NCCL (after timing)
    gather_ms = None
    n_rings_total = int(counts.clamp(min=0).sum().item())
    if world > 1:
        from paper_1310_1371_b200.distributed import gather_rings
        torch.cuda.synchronize(dev)
        g0 = time.perf_counter()
        res = gather_rings(rings, counts)
        torch.cuda.synchronize(dev)
        gather_ms = (time.perf_counter() - g0) * 1e3
        if res is not None:
            n_rings_total = int(res[1].clamp(min=0).sum().item())

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---------------- roofline of the dominant kernel
    names = ["k_ridges", "k_rays", "k_hough", "k_fit"]
    kms_all = [k / ncalls for k in kms]
    kms_step = [kms_all[0], kms_all[2], kms_all[3]]      # K1, K2, K3 (K1.5 reported separately)
    dom = int(np.argmax(kms_step))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    # K1: fp64 pipe (exact stencil arithmetic); peak = 148 SM x 64 DFMA/clk x sm_max
    Ks = math.ceil(3 * params["smoothing_sigma"])
    k1_ops_per_px = (2 * Ks + 1) + 9 + 9 + 10
    px = params["width"] * params["height"]
    fp64_peak = 148 * 64 * sm_max * 1e6 / 1e12
    k1_ach = B * px * k1_ops_per_px / (kms_step[0] / 1e3) / 1e12
    # K2: one shared-memory atomic per in-frame vote is the irreducible work of an
    # accumulator Hough transform; peak = measured ATOMS throughput 11.0/clk/SM
    # (tools/microbench, profiles/microbench_r01.log) x 148 SM x sm_max
    atom_peak = 11.0 * 148 * sm_max * 1e6 / 1e9
    k2_ach = votes_per_step / (kms_step[1] / 1e3) / 1e9
    # K2 as an ALU-issue-bound kernel: algorithmic lane operations per frame =
    # 11 per in-frame vote (~10 ops + 1 atomic) + 2 per hotspot window cell
    # (multiply-add); the NMS compares (<1 %) are left out; peak = 148 SM x 128 lanes x sm_max
    k2_ops = 11 * votes_per_step + 2 * win_cells_per_frame * B
    lane_peak = 148 * 128 * sm_max * 1e6 / 1e12
    k2_alu = k2_ops / (kms_step[1] / 1e3) / 1e12
    summ = {}
    sp = os.path.join(ROOT, "profiles", "ncu_summary_r01.json")
    if os.path.exists(sp):
        for d in json.load(open(sp)):
            for n in names:
                if n in d.get("kernel", "") and "dram_bytes_per_frame" in d:
                    summ[n] = d["dram_bytes_per_frame"] * B
    roofs = [
        {"kernel": "k_ridges", "bound": "alu", "achieved": round(k1_ach, 3), "peak": round(fp64_peak, 3),
         "unit": "TFLOP/s", "frac": round(k1_ach / fp64_peak, 4), "traffic": summ.get("k_ridges"),
         "peak_note": "fp64 DFMA issue: 148 SM x 64/clk x sm_max (guide unit counts); ops = fp64 instructions of "
                      "the exact separable Gaussian + Sobel + kappa per pixel (DESIGN.md §6)"},
        {"kernel": "k_hough", "bound": "alu", "achieved": round(k2_alu, 4), "peak": round(lane_peak, 2),
         "unit": "T lane-op/s", "frac": round(k2_alu / lane_peak, 5), "traffic": summ.get("k_hough"),
         "peak_note": "ALU issue: 148 SM x 128 lanes x sm_max (guide unit counts); ops = 11 per in-frame vote + "
                      "2 per hotspot window cell (SURVEY.md §8(d), DESIGN.md §6); window cells "
                      f"{win_cells_per_frame:.0f}/frame measured by a debug pass"},
        {"kernel": "k_hough", "bound": "alu", "achieved": round(k2_ach, 3), "peak": round(atom_peak, 1),
         "unit": "Gvote/s", "frac": round(k2_ach / atom_peak, 5), "traffic": summ.get("k_hough"),
         "peak_note": "shared-memory atomic issue: measured 11.0 ATOMS/clk/SM x 148 SM x sm_max; one atomic per "
                      "in-frame vote (DESIGN.md §6)"},
    ]
    roof = dict(roofs[0] if dom == 0 else roofs[1])
    hbm_peak = float(peaks.get("hbm_gbs", 6549.1))
    alg_bytes_frame = fbytes + 64 * (n_rings_total / max(1, B * world))
    hbm_achieved = alg_bytes_frame * value / world / 1e9

    cpu = None
    if world == 1 and not args.no_cpu:
        n_cpu = args.cpu_frames
        rate, cores, dt = cpu_oracle_rate(n_cpu, frames=frames_h[:n_cpu])
        cpu = {"value": round(rate, 3), "unit": "frames/s", "cores": cores, "kind": "oracle",
               "sample": f"first {n_cpu} frames of this batch (cfg3, full frames), {dt:.1f} s wall"}
        srate, _, sdt = cpu_oracle_rate(n_cpu, frames=frames_h[:n_cpu], streamed=True)
        cpu["paper_streamed"] = {"value": round(srate, 3), "unit": "frames/s", "cores": cores,
                                 "note": "the paper's streamed CPU method (sorted vote stack, r mod 3 "
                                         f"sub-spaces; oracle/streamed.c), same sample, {sdt:.1f} s wall"}

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
            "e2e": {"value": round(e2e_value, 1), "unit": "frames/s", "steps": e2e_steps,
                    "h2d_bytes_per_step": B * fbytes * world,
                    "d2h_bytes_per_step": (B * det.ring_cap * 64 + 4 * B) * world,
                    "api": "Detector.detect_host -> rd_detect_host (pinned host buffers)"},
            # K1, K1.5, K2, K2 redo reset, K2 redo pass, K3 per batch; a batch of >= 128 frames
            # runs as two halves
            "gpu_launches": 6 * (2 if B >= 128 else 1) * args.steps,
            "clocks": clocks}
    if gather_ms is not None:
        line["gather_ms"] = round(gather_ms, 3)
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
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-frames", type=int, default=256)
    ap.add_argument("--ref-frames", type=int, default=32)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
