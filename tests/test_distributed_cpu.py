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


# --- the frame-group protocol (distributed.FrameGroup) over gloo ----------------------


class _ShmGroup:
    """Stand-in for csrc/vx_group.cu with the same five calls: rank 0's two
    frame slots live in a shared file; a rank's render stores its owned
    tiles there and adds its counters under a lock (the native group does
    this with peer stores and system-scope atomics), using the CPU oracle
    for the pixels."""

    def __init__(self, workdir, volume, T):
        self.dir, self.volume, self.T = workdir, volume, T

    def create(self, rank, world, max_pixels):
        self.rank, self.world, self.max_pixels = rank, world, max_pixels
        self.frame = self.released = 0
        return f"{self.dir}/slots.bin".encode()

    def shares_device(self, group):
        return True

    def connect(self, blobs, sync):
        import fcntl

        path = blobs[: len(blobs) // self.world].decode()  # rank 0's blob: its slot file
        if self.rank == 0:
            np.zeros(2 * (self.max_pixels + 259 * 8), np.uint8).tofile(path)
        import torch.distributed as dist

        dist.barrier()
        self.mm = np.memmap(path, dtype=np.uint8, mode="r+")
        self.lock = open(path + ".lock", "w")
        self._fcntl = fcntl
        return sync

    def _slot(self, f):
        off = (f & 1) * (self.max_pixels + 259 * 8)
        return self.mm[off:off + self.max_pixels], self.mm[off + self.max_pixels:
                                                         off + self.max_pixels + 259 * 8].view(np.uint64)

    def render(self, dvol, rs, rp, fc, stream):
        from oracle import oracle as orc
        from paper_1807_03119_b200.distributed import owned_pixel_mask

        cam, W, H = rs
        self.frame += 1
        full = orc.render(self.volume, cam, W, H, kind="local-cluster", threshold=self.T)
        mask = owned_pixel_mask(W, H, self.rank, self.world)
        pix, cnt = self._slot(self.frame)
        self._fcntl.flock(self.lock, self._fcntl.LOCK_EX)
        flat = pix[:W * H]
        flat[mask.reshape(-1)] = full["pixels"].reshape(-1)[mask.reshape(-1)]
        cnt[:256] += np.bincount(full["pixels"][mask], minlength=256).astype(np.uint64)
        cnt[256] += np.uint64(int((full["hit_voxel"][:, 0] >= 0)[mask.reshape(-1)].sum()))
        self.mm.flush()
        self._fcntl.flock(self.lock, self._fcntl.LOCK_UN)
        return self.frame

    def download(self, pixels, counters, stream):
        pix, cnt = self._slot(self.released + 1)
        pixels.reshape(-1)[:] = pix[:pixels.size]
        counters[:259] = cnt.view(np.int64)

    def release(self, stream):
        self.released += 1
        self._slot(self.released)[1][:] = 0

    def close(self):
        pass


def _group_worker(rank, world, port, workdir, q):
    import sys

    sys.path.insert(0, os.getcwd())
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_1807_03119_b200.distributed import FrameGroup

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rs = np.random.default_rng(1)
        vol = rs.integers(0, 60, (29, 23, 31), dtype=np.uint8)
        vol[8:20, 6:16, 9:22] = 190
        T = float(orc.otsu(orc.hist256(vol)))
        W, H = 43, 35
        fg = FrameGroup(W * H, backend=_ShmGroup(workdir, vol, T))
        assert fg.host_sync
        ok = True
        for k, az in enumerate((10.0, 100.0, 230.0, 300.0)):
            pos, look = orc.orbit((31, 23, 29), azimuth_deg=az)
            cam = orc.cam_vector(pos, look, W, H)
            fg.render(None, (cam, W, H), None, None, 0)
            fg.finish()
            if rank == 0:
                full = orc.render(vol, cam, W, H, kind="local-cluster", threshold=T)
                pix = np.zeros((H, W), np.uint8)
                cnt = np.zeros(266, np.int64)
                fg.download(pix, cnt, 0)
                fg.release(0)
                ok &= np.array_equal(pix, full["pixels"])
                ok &= np.array_equal(cnt[:256], np.bincount(full["pixels"].reshape(-1),
                                                            minlength=256))
                ok &= int(cnt[256]) == full["hit_count"]
        q.put((rank, bool(ok), fg.frames))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_frame_group_protocol(world, tmp_path):
    """FrameGroup over gloo: blob exchange, host-ordered frames, slot reuse
    (four frames through two slots), rank 0's download and release."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_group_worker, args=(r, world, port, str(tmp_path), q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    assert all(n == 4 for *_, n in res)


class _FlakyGroup:
    """Backend whose device-flag connect fails on rank 1 (e.g. no stream
    memops across a peer mapping): every rank must end up host-ordered."""

    def create(self, rank, world, max_pixels):
        self.rank = rank
        return b"x"

    def shares_device(self, group):
        return False

    def probe_device_sync(self):
        return True

    def connect(self, blobs, sync):
        from paper_1807_03119_b200 import _lib

        if sync == _lib.VX_GROUP_SYNC_DEVICE and self.rank == 1:
            raise _lib.NativeError(3, "peer flag probe failed (CUresult 801)")
        return sync

    def close(self):
        pass


def _fallback_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.getcwd())
    import torch.distributed as dist

    from paper_1807_03119_b200 import _lib
    from paper_1807_03119_b200.distributed import FrameGroup

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fg = FrameGroup(100, backend=_FlakyGroup())
        q.put((rank, fg.sync == _lib.VX_GROUP_SYNC_HOST, fg.host_sync))
    finally:
        dist.destroy_process_group()


def test_gloo_frame_group_falls_back_to_host_ordering():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(host and hs for _, host, hs in res)
