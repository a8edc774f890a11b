"""Frame sharding and ring-list collection across ranks (one process per GPU).

The method has no cross-frame state (frames are analysed by independent
worker processes in a producer/consumer scheme), so frames are split into contiguous
ranges per rank and the only collective is the final gather of the per-frame ring
lists to rank 0 (torch.distributed: NCCL on GPUs, gloo on CPU).  No accumulator, ridge
or halo ever crosses ranks.  This module is plumbing around the C ABI: the detection
itself runs in librd.so.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from ._rd import RING_DTYPE

REC = RING_DTYPE.itemsize  # 64 bytes per ring record


def shard(n_frames: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous frame range [start, end) of `rank`; sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world) or n_frames < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def pack(rings: torch.Tensor, counts: torch.Tensor, offsets: torch.Tensor | None = None):
    """Dense records of a detect call: (records [total, 64] uint8 in frame order, canonical order
    within a frame; counts int64 with -1 for overflowed frames).  rings is either rd_detect's
    compact buffer [capacity, 64] with its offsets, or a padded [n, cap, 64] buffer (offsets None)."""
    c = counts.to(torch.int64)
    valid = c.clamp(min=0)
    if offsets is None:
        n, cap = rings.shape[0], rings.shape[1]
        mask = torch.arange(cap, device=rings.device).unsqueeze(0) < valid.unsqueeze(1)
        return rings[mask].reshape(-1, REC), c
    # compact: the valid frames' rings are back to back unless a frame with count -1 left a hole
    # (output capacity); then gather the valid ranges
    cc = c.cpu()
    if bool((cc >= 0).all()):
        return rings.reshape(-1, REC)[: int(cc.sum())], c
    o = offsets[:-1].to(torch.int64)
    total = int(valid.sum())
    if total == 0:
        return torch.zeros((0, REC), dtype=torch.uint8, device=rings.device), c
    frame = torch.repeat_interleave(torch.arange(len(c), device=rings.device), valid)
    first = torch.cumsum(valid, 0) - valid
    idx = o[frame] + (torch.arange(total, device=rings.device) - first[frame])
    return rings.reshape(-1, REC)[idx], c


def gather_rings(rings: torch.Tensor, counts: torch.Tensor, offsets: torch.Tensor | None = None, dst: int = 0,
                 group=None):
    """Gather every rank's rings to `dst`: an all_gather of the per-rank sizes,
    then one gather to dst of the records padded to the largest rank (only dst receives P
    buffers).  Returns, on dst, (records [N_total, 64] uint8 in rank order, counts
    [n_frames_total] int64 with -1 for overflowed frames); None elsewhere."""
    return gather_records(*pack(rings, counts, offsets), dst=dst, group=group)


def gather_records(recs: torch.Tensor, cnt: torch.Tensor, dst: int = 0, group=None):
    """gather_rings on already packed records ([total, 64] uint8, int64 counts per frame)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = recs.device
    sizes = torch.tensor([recs.shape[0], cnt.shape[0]], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    max_r = max(int(s[0]) for s in all_sizes)
    max_f = max(int(s[1]) for s in all_sizes)
    # one buffer per rank: frame counts (int64) then the records, as bytes
    cb = max(max_f, 1) * 8
    buf = torch.zeros(cb + max(max_r, 1) * REC, dtype=torch.uint8, device=dev)
    cpad = torch.full((max(max_f, 1),), -2, dtype=torch.int64, device=dev)
    cpad[: cnt.shape[0]] = cnt
    buf[:cb] = cpad.view(torch.uint8)
    buf[cb:cb + recs.numel()] = recs.reshape(-1)
    gl = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, gl, dst=dst, group=group)
    if rank != dst:
        return None
    out_r = torch.cat([gl[i][cb:cb + int(all_sizes[i][0]) * REC].reshape(-1, REC) for i in range(world)])
    out_c = torch.cat([gl[i][:cb].view(torch.int64)[: int(all_sizes[i][1])] for i in range(world)])
    return out_r, out_c


def collect(batches, dst: int = 0, group=None):
    """The multi-GPU result path of SURVEY.md §8(e) (bench.py --config 5): this rank's detect
    outputs (a list of (rings, counts, offsets) in frame order, compact or padded) are packed and
    gathered to `dst`.  Returns (records [N_total, 64] uint8, counts int64) on dst — in rank order,
    so byte-identical for every world size when ranks hold contiguous frame ranges — None on the
    other ranks.  Without an initialised process group the local lists are returned."""
    batches = list(batches)
    if batches and all(len(b) == 3 and b[2] is not None for b in batches):
        # compact outputs: one host read of all counts; with no overflowed frame every batch's
        # records are the prefix of its buffer (no per-batch synchronisation)
        cnts = torch.cat([b[1].to(torch.int64) for b in batches])
        hc = cnts.cpu()
        if bool((hc >= 0).all()):
            sizes, pos = [], 0
            for b in batches:
                n = b[1].shape[0]
                sizes.append(int(hc[pos:pos + n].sum()))
                pos += n
            recs = torch.cat([b[0].reshape(-1, REC)[:m] for b, m in zip(batches, sizes)])
            if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
                return recs, cnts
            return gather_records(recs, cnts, dst=dst, group=group)
    packed = [pack(*b) for b in batches]
    if packed:
        recs = torch.cat([p[0] for p in packed])
        cnts = torch.cat([p[1] for p in packed])
    else:
        recs, cnts = torch.zeros((0, REC), dtype=torch.uint8), torch.zeros(0, dtype=torch.int64)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return recs, cnts
    return gather_records(recs, cnts, dst=dst, group=group)


def digest(records: torch.Tensor, counts: torch.Tensor) -> str:
    """sha256 of gathered records and counts (the P-invariance check of SURVEY.md §4 T4)."""
    import hashlib
    return hashlib.sha256(records.cpu().numpy().tobytes() + counts.cpu().numpy().astype(np.int64).tobytes()).hexdigest()


def unpack(records: torch.Tensor, counts: torch.Tensor) -> list:
    """Per-frame structured arrays (RING_DTYPE) from packed records; None for overflowed frames."""
    arr = records.cpu().numpy().reshape(-1).view(RING_DTYPE)
    out, pos = [], 0
    for c in counts.cpu().numpy().tolist():
        if c < 0:
            out.append(None)
            continue
        out.append(arr[pos:pos + c].copy())
        pos += c
    return out


__all__ = ["shard", "pack", "gather_rings", "gather_records", "collect", "digest", "unpack", "REC"]
