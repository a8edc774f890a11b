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


def pack(rings: torch.Tensor, counts: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Compact a [n, cap, 64] uint8 ring buffer with per-frame counts into contiguous records
    [total, 64] uint8 (frame order, canonical order within a frame) + counts (int64)."""
    n, cap = rings.shape[0], rings.shape[1]
    c = counts.to(torch.int64).clamp(min=0)
    mask = torch.arange(cap, device=rings.device).unsqueeze(0) < c.unsqueeze(1)
    return rings[mask].reshape(-1, REC), counts.to(torch.int64)


def gather_rings(rings: torch.Tensor, counts: torch.Tensor, dst: int = 0, group=None):
    """Gather every rank's rings to `dst`.  Returns, on dst, (records [N_total, 64] uint8 in
    rank order, counts [n_frames_total] int64 with -1 for overflowed frames); None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    recs, cnt = pack(rings, counts)
    dev = recs.device
    sizes = torch.tensor([recs.shape[0], cnt.shape[0]], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    max_r = max(int(s[0]) for s in all_sizes)
    max_f = max(int(s[1]) for s in all_sizes)
    pr = torch.zeros((max(max_r, 1), REC), dtype=torch.uint8, device=dev)
    pr[: recs.shape[0]] = recs
    pc = torch.full((max(max_f, 1),), -2, dtype=torch.int64, device=dev)
    pc[: cnt.shape[0]] = cnt
    gr = [torch.empty_like(pr) for _ in range(world)]
    gc = [torch.empty_like(pc) for _ in range(world)]
    dist.all_gather(gr, pr, group=group)
    dist.all_gather(gc, pc, group=group)
    if rank != dst:
        return None
    out_r = torch.cat([gr[i][: int(all_sizes[i][0])] for i in range(world)])
    out_c = torch.cat([gc[i][: int(all_sizes[i][1])] for i in range(world)])
    return out_r, out_c


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


__all__ = ["shard", "pack", "gather_rings", "unpack", "REC"]
_ = np  # numpy is used through RING_DTYPE views
