"""Multi-rank host logic on CPU (gloo, world_size 2): z-slab histogram sharding
+ all-reduce, sort-first tile partition + frame reduce.  The per-rank compute
is the CPU oracle here (the B200 kernels are exercised by the gpu tests)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.getcwd())
    import torch
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_1807_03119_b200.distributed import (allreduce_counts, owned_pixel_mask,
                                                   reduce_frame, slab_bounds)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rs = np.random.default_rng(0)
        vol = rs.integers(0, 60, (37, 21, 19), dtype=np.uint8)
        vol[10:25, 5:15, 4:14] = 200
        # histogram: each rank counts its slab, bins are all-reduced
        z0, z1 = slab_bounds(vol.shape[0], rank, world)
        counts = allreduce_counts(orc.hist256(vol[z0:z1]))
        ok_hist = np.array_equal(counts.numpy(), np.bincount(vol.reshape(-1), minlength=256))
        T = orc.otsu(counts.numpy())
        # frame: each rank contributes its owned tiles, summed onto rank 0
        W, H = 45, 37
        pos, look = orc.orbit((19, 21, 37))
        cam = orc.cam_vector(pos, look, W, H)
        full = orc.render(vol, cam, W, H, kind="local-cluster", threshold=float(T))["pixels"]
        part = np.where(owned_pixel_mask(W, H, rank, world), full, 0).astype(np.uint8)
        t = torch.from_numpy(part.reshape(-1).copy())
        reduce_frame(t, 0)
        ok_frame = True if rank != 0 else np.array_equal(t.numpy().reshape(H, W), full)
        q.put((rank, ok_hist, ok_frame, T))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_histogram_and_frame_reduce(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok_h and ok_f for _, ok_h, ok_f, _ in res)
    assert len({T for *_, T in res}) == 1  # identical Otsu T on every rank


def test_partition_helpers():
    from paper_1807_03119_b200.distributed import owned_pixel_mask, slab_bounds

    for world in (1, 2, 3, 4, 8):
        masks = [owned_pixel_mask(61, 45, r, world) for r in range(world)]
        assert np.array_equal(sum(m.astype(int) for m in masks), np.ones((45, 61), int))
        spans = [slab_bounds(1000, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 1000
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
