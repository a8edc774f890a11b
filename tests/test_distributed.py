"""Multi-process frame sharding and ring gathering on CPU (gloo, world_size 2) (-m "not gpu").

The GPU run uses the same code over NCCL (bench.py --gpus N under torchrun).  Per-rank
ring lists here come from the CPU oracle (test infrastructure), so the test checks the
sharding + gather plumbing: the gathered lists equal a single-process run, byte for byte,
for every world size and shard split (test tier T4).
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1310_1371_b200 import distributed as D
from paper_1310_1371_b200._rd import RING_DTYPE

CAP = 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rings_buffer(ring_lists):
    buf = np.zeros((len(ring_lists), CAP), dtype=RING_DTYPE)
    counts = np.zeros(len(ring_lists), dtype=np.int32)
    for i, r in enumerate(ring_lists):
        if r is None:
            counts[i] = -1
            continue
        buf[i, : len(r)] = r.view(RING_DTYPE)
        counts[i] = len(r)
    return torch.from_numpy(buf.view(np.uint8).reshape(len(ring_lists), CAP, 64).copy()), torch.from_numpy(counts)


def _worker(rank, world, port, n_frames, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = oracle.params(**synth.preset(2))
    a, b = D.shard(n_frames, world, rank)
    frames = synth.batch(2, 0, a, b - a) if b > a else np.zeros((0, 480, 640), np.uint8)
    lists = [oracle.detect(p, f)[0] for f in frames]
    if rank == 1 and len(lists) > 0:
        lists[0] = None  # an overflowed frame travels as count -1
    rings, counts = _rings_buffer(lists) if lists else (torch.zeros((0, CAP, 64), dtype=torch.uint8),
                                                         torch.zeros(0, dtype=torch.int32))
    res = D.gather_rings(rings, counts)
    if rank == 0:
        recs, cnt = res
        torch.save({"recs": recs, "counts": cnt}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_partitions():
    for n in (0, 1, 7, 16, 8192):
        for w in (1, 2, 3, 4, 8):
            ranges = [D.shard(n, w, r) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.shard(4, 2, 2)


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(0)
    lists = []
    for n in (3, 0, 5, 1):
        a = np.zeros(n, dtype=RING_DTYPE)
        a["cx"] = rng.integers(0, 100, n)
        a["fx"] = rng.normal(size=n)
        lists.append(a)
    lists.append(None)
    rings, counts = _rings_buffer(lists)
    recs, cnt = D.pack(rings, counts)
    assert recs.shape == (9, 64) and cnt.tolist() == [3, 0, 5, 1, -1]
    back = D.unpack(recs, cnt)
    for a, b in zip(lists, back):
        assert (a is None and b is None) or a.tobytes() == b.tobytes()


@pytest.mark.parametrize("world,n_frames", [(2, 5), (2, 1)])
def test_gather_gloo_matches_single_process(world, n_frames):
    port = _free_port()
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "g.pt")
        mp.spawn(_worker, args=(world, port, n_frames, out), nprocs=world, join=True)
        got = torch.load(out)
    p = oracle.params(**synth.preset(2))
    frames = synth.batch(2, 0, 0, n_frames)
    expect = [oracle.detect(p, f)[0] for f in frames]
    a1, _ = D.shard(n_frames, world, 1)
    if a1 < n_frames:
        expect[a1] = None
    back = D.unpack(got["recs"], got["counts"])
    assert len(back) == n_frames
    for e, g in zip(expect, back):
        assert (e is None and g is None) or e.view(RING_DTYPE).tobytes() == g.tobytes()


# ---------------------------------------------------------------- bench.py --config 5 path
def _compact(ring_lists, cap_extra=3):
    """rd_detect-style compact output of per-frame lists: rings back to back (a frame with
    None overflowed: count -1, no rings), counts, CSR offsets."""
    counts = np.array([-1 if r is None else len(r) for r in ring_lists], dtype=np.int32)
    offsets = np.zeros(len(ring_lists) + 1, dtype=np.int32)
    offsets[1:] = np.cumsum(np.maximum(counts, 0))
    buf = np.zeros(offsets[-1] + cap_extra, dtype=RING_DTYPE)
    for i, r in enumerate(ring_lists):
        if r is not None:
            buf[offsets[i]:offsets[i + 1]] = r.view(RING_DTYPE)
    return (torch.from_numpy(buf.view(np.uint8).reshape(-1, 64).copy()), torch.from_numpy(counts),
            torch.from_numpy(offsets))


def _sweep_worker(rank, world, port, n_frames, batch, out_path):
    """One rank of the cfg5 sweep (bench.run_sweep's result path): its contiguous frame range
    in batches, detected (here by the oracle), collected to rank 0."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = oracle.params(**synth.preset(2))
    a, b = D.shard(n_frames, world, rank)
    batches = []
    for s in range(a, b, batch):
        lists = [oracle.detect(p, f)[0] for f in synth.batch(2, 0, s, min(batch, b - s))]
        if s == a and rank == world - 1:
            lists[0] = None   # an overflowed frame travels as count -1
        batches.append(_compact(lists))
    res = D.collect(batches)
    if rank == 0:
        torch.save({"recs": res[0], "counts": res[1], "digest": D.digest(*res)}, out_path)
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sweep_collect_invariant_to_world_size(world):
    """the gathered cfg5-style lists are byte-identical (same sha256) for every
    world size and equal the single-process lists frame by frame."""
    n_frames, batch = 7, 3
    port = _free_port()
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "s.pt")
        mp.spawn(_sweep_worker, args=(world, port, n_frames, batch, out), nprocs=world, join=True)
        got = torch.load(out)
    p = oracle.params(**synth.preset(2))
    expect = [oracle.detect(p, f)[0] for f in synth.batch(2, 0, 0, n_frames)]
    expect[D.shard(n_frames, world, world - 1)[0]] = None
    ref = D.collect([_compact(expect[s:s + batch]) for s in range(0, n_frames, batch)])   # one process
    assert D.digest(*ref) != "" and got["recs"].numel() > 0
    back = D.unpack(got["recs"], got["counts"])
    for e, g in zip(expect, back):
        assert (e is None and g is None) or e.view(RING_DTYPE).tobytes() == g.tobytes()
    # byte identity with the single-process collect (the None frame sits at the same index)
    assert torch.equal(got["recs"], ref[0]) and torch.equal(got["counts"], ref[1])
    assert got["digest"] == D.digest(*ref)

