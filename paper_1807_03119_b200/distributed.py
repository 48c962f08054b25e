"""Multi-GPU plumbing: one process per GPU, torch.distributed for set-up.

Sort-first parallel rendering, the reference's worker split
(render.py:514-541: row bands on a thread pool, bit-identical for any worker
count, test_render.py:242-251) at GPU granularity:

* **Volume.** Every rank holds the full replica.  ``replicate_volume`` loads
  or generates it once on the source rank and broadcasts the compact bytes
  (NCCL over NVLink on the B200 box); every rank then builds its padded
  replica and skip maps from them on its own device.
* **Histogram / Otsu.** Each rank counts the contiguous z-slab
  ``slab_bounds(nz, rank, world)`` *of the replica it already holds*
  (``vx_volume_histogram_slab``), the 256 u64 bins are all-reduced (2 KiB),
  and every rank runs the exact K2 scan on the sum: identical T everywhere.
* **Frames.** 8x16 tiles are dealt round-robin (tile t -> rank t % world) so
  early-terminating hit rays and long miss rays balance.  There is no
  collective per frame: every rank's K4 stores its tiles straight into rank
  0's frame slot through a peer (CUDA-IPC) pointer and adds the image
  histogram / hit count there with system-scope atomics; completion and slot
  reuse are monotonic flags written and awaited with stream memory
  operations (csrc/vx_group.cu).  Ranks that share one GPU (the functional
  mode of a one-GPU box) order frames on the host instead: stream sync and a
  barrier per frame.

Per-frame communication at N ranks: each rank writes its ~1/N of the W*H
pixel bytes over NVLink as part of its own kernel, plus <= 256 + 2 counter
atomics per warp-tile; rank 0 waits on N - 1 flags; release writes N - 1
flags.  No NCCL launch, no full-frame zeroing, no reduction of zeros.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib

TILE_W, TILE_H = 8, 16  # csrc/vx_render.cu kTileW / kTileH


def slab_bounds(nz: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous z-planes [z0, z1) of rank's slab: ceil(nz/world) planes each."""
    per = -(-nz // world)
    z0 = min(nz, rank * per)
    return z0, min(nz, z0 + per)


def owned_pixel_mask(width: int, height: int, rank: int, world: int) -> np.ndarray:
    """(H, W) bool mask of the pixels rank renders (the kernel's tile deal)."""
    tiles_x = -(-width // TILE_W)
    j, i = np.mgrid[0:height, 0:width]
    tile = (j // TILE_H) * tiles_x + (i // TILE_W)
    return (tile % world) == rank


def allreduce_counts(counts, group=None):
    """Sum 256-bin histograms across ranks (the 2 KiB all-reduce)."""
    import torch
    import torch.distributed as dist

    t = counts if isinstance(counts, torch.Tensor) else torch.as_tensor(
        np.asarray(counts, dtype=np.int64))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def reduce_frame(pixels, dst: int = 0, group=None):
    """Sum partial frames (zero outside owned tiles) onto dst.  Host-side
    reference of the tile deal, used by the CPU tests; the device path writes
    tiles into rank 0's slot instead (FrameGroup)."""
    import torch.distributed as dist

    dist.reduce(pixels, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return pixels


def all_gather_bytes(blob: bytes, group=None) -> list[bytes]:
    """Every rank's blob, in rank order (the C-ABI group's address exchange)."""
    import torch.distributed as dist

    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    return [bytes(b) for b in out]


def shares_device(group=None) -> bool:
    """True when two ranks of the group drive the same GPU (one-GPU box)."""
    import torch
    import torch.distributed as dist

    uuid = str(torch.cuda.get_device_properties(torch.cuda.current_device()).uuid)
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, uuid, group=group)
    return len(set(out)) < len(out)


# --- the native frame group (C-ABI vx_group_*) --------------------------------------


class NativeGroup:
    """ctypes face of csrc/vx_group.cu (one per rank)."""

    def __init__(self):
        self.handle = C.c_void_p()

    def create(self, rank: int, world: int, max_pixels: int) -> bytes:
        _lib.require_device()
        blob = np.zeros(_lib.VX_GROUP_BLOB_BYTES, dtype=np.uint8)
        _lib.call("vx_group_create", rank, world, int(max_pixels), C.byref(self.handle),
                  _lib.ptr(blob))
        return blob.tobytes()

    def probe_device_sync(self) -> bool:
        return _lib.load().vx_group_probe_device_sync() == _lib.VX_OK

    def connect(self, blobs: bytes, sync: int) -> int:
        buf = np.frombuffer(blobs, dtype=np.uint8).copy()
        _lib.call("vx_group_connect", self.handle, _lib.ptr(buf), int(sync))
        mode = C.c_int32(-2)
        _lib.call("vx_group_info", self.handle, C.byref(mode), None)
        return int(mode.value)

    def render(self, dvol, rs, rp, fc, stream: int):
        out = _lib.vx_group_frame()
        _lib.call("vx_group_render", self.handle, dvol.handle, C.byref(rs), C.byref(rp),
                  C.byref(fc), C.c_void_p(stream), C.byref(out))
        return out

    def download(self, pixels: np.ndarray, counters: np.ndarray, stream: int) -> None:
        _lib.call("vx_group_download", self.handle, _lib.ptr(pixels), _lib.ptr(counters),
                  pixels.size, C.c_void_p(stream))

    def release(self, stream: int) -> None:
        _lib.call("vx_group_release", self.handle, C.c_void_p(stream))

    def close(self) -> None:
        if self.handle:
            _lib.load().vx_group_destroy(self.handle)
            self.handle = C.c_void_p()


class FrameGroup:
    """Sort-first frame exchange of a process group (see the module docstring).

    Per frame every rank calls ``render`` then ``finish``; rank 0 then
    consumes the frame (``download`` or the device pointers ``render``
    returned) and calls ``release``.  ``backend`` is the native group, or a
    stand-in with the same five methods (the CPU tests drive the protocol
    with the oracle).
    """

    def __init__(self, max_pixels: int, group=None, sync: str = "auto", backend=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.max_pixels = int(max_pixels)
        self.backend = backend if backend is not None else NativeGroup()
        if sync == "auto":
            # decided collectively: every rank must agree on the protocol
            mode = (_lib.VX_GROUP_SYNC_HOST if self._shared(group) or not self._memops_ok(group)
                    else _lib.VX_GROUP_SYNC_DEVICE)
        else:
            mode = {"device": _lib.VX_GROUP_SYNC_DEVICE, "host": _lib.VX_GROUP_SYNC_HOST}[sync]
        self.sync = self._setup(mode, group)
        self.frames = 0

    def _setup(self, mode: int, group) -> int:
        """create, all-gather the blobs, connect.  If the device flags fail
        on any rank (connect probes them across the peer mappings), every
        rank rebuilds its group with host ordering."""
        import torch.distributed as dist

        blob = self.backend.create(self.rank, self.world, self.max_pixels)
        blobs = all_gather_bytes(blob, group)
        try:
            got, ok = self.backend.connect(b"".join(blobs), mode), True
        except _lib.NativeError:
            if mode != _lib.VX_GROUP_SYNC_DEVICE:
                raise
            got, ok = None, False
        flags: list = [None] * self.world
        dist.all_gather_object(flags, ok, group=group)
        if all(flags):
            return got
        self.backend.close()
        self.backend = type(self.backend)()
        return self._setup(_lib.VX_GROUP_SYNC_HOST, group)

    def _memops_ok(self, group) -> bool:
        """Every rank's device supports the stream-memop flags."""
        import torch.distributed as dist

        probe = getattr(self.backend, "probe_device_sync", None)
        ok = probe() if probe is not None else True
        out: list = [None] * self.world
        dist.all_gather_object(out, bool(ok), group=group)
        return all(out)

    def _shared(self, group) -> bool:
        shared = getattr(self.backend, "shares_device", None)
        return shared(group) if shared is not None else shares_device(group)

    @property
    def host_sync(self) -> bool:
        return self.sync == _lib.VX_GROUP_SYNC_HOST and self.world > 1

    def render(self, dvol, rs, rp, fc, stream: int):
        """This rank's tiles of the next frame (asynchronous on ``stream``)."""
        out = self.backend.render(dvol, rs, rp, fc, stream)
        self.frames += 1
        return out

    def finish(self, stream_obj=None) -> None:
        """Host-ordered mode: every rank's tiles are in before anyone goes on."""
        if not self.host_sync:
            return
        import torch.distributed as dist

        if stream_obj is not None:
            stream_obj.synchronize()
        dist.barrier(group=self.group)

    def download(self, pixels: np.ndarray, counters: np.ndarray, stream: int) -> None:
        self.backend.download(pixels, counters, stream)

    def release(self, stream: int) -> None:
        if self.rank == 0:
            self.backend.release(stream)

    def close(self) -> None:
        self.backend.close()


# --- volume replication and the sharded histogram ------------------------------------


def replicate_volume(dims, group=None, src: int = 0, volume=None, fill=None):
    """DeviceVolume replica on every rank from one source: the compact bytes
    come from ``volume`` (a host Volume) or ``fill(tensor)`` (e.g. the device
    phantom generator) on rank ``src`` and are broadcast to the others."""
    import torch
    import torch.distributed as dist

    from .volume import DeviceVolume, VolumeError

    nx, ny, nz = (int(d) for d in dims)
    dev = torch.device("cuda", torch.cuda.current_device())
    compact = torch.empty(nx * ny * nz, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == src:
        if volume is not None:
            compact.copy_(torch.from_numpy(np.ascontiguousarray(volume.data).reshape(-1)))
        elif fill is not None:
            fill(compact)
        else:
            raise ValueError("the source rank needs a volume or a fill function")
    dist.broadcast(compact, src=src, group=group)
    torch.cuda.current_stream(dev).synchronize()
    h = C.c_void_p()
    _lib.call("vx_volume_create_device_u8", C.c_void_p(compact.data_ptr()), nx, ny, nz,
              C.byref(h), exc_type=VolumeError)
    del compact
    return DeviceVolume(h, (nx, ny, nz))


def histogram_sharded(volume, group=None):
    """HistogramModel from z-slabs of the replica (K1 per slab + all-reduce + K2).

    ``volume`` is a Volume (its cached replica is used) or a DeviceVolume.
    """
    import torch
    import torch.distributed as dist

    from .histogram import model_from_counts
    from .volume import DeviceVolume, device_volume

    dv = volume if isinstance(volume, DeviceVolume) else device_volume(volume)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    z0, z1 = slab_bounds(dv.dims[2], rank, world)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    counts = torch.zeros(256, dtype=torch.int64, device=dev)
    _lib.call("vx_volume_histogram_slab", dv.handle, z0, z1, C.c_void_p(counts.data_ptr()),
              C.c_void_p(stream.cuda_stream))
    allreduce_counts(counts, group)
    return model_from_counts(counts.cpu().numpy())


# --- one frame over the group ----------------------------------------------------------

_groups: dict = {}


def frame_group(max_pixels: int, group=None) -> FrameGroup:
    """The cached FrameGroup of (process group, frame size) (collective on first use)."""
    key = (id(group), int(max_pixels))
    fg = _groups.get(key)
    if fg is None:
        fg = _groups[key] = FrameGroup(max_pixels, group)
    return fg


def render_sharded(volume, camera, params, config, histogram=None, group=None,
                   fgroup: FrameGroup | None = None):
    """Render one frame split over the group's GPUs; rank 0 gets the Frame,
    the other ranks None.  Collective: every rank calls it for every frame."""
    import torch

    from .render import Frame, _check_render_args, _native, render_detail
    from .volume import DeviceVolume, device_volume

    wall0 = time.perf_counter()
    config = _check_render_args(config, histogram, None)
    dv = volume if isinstance(volume, DeviceVolume) else device_volume(volume)
    W, H = params.width, params.height
    fg = fgroup if fgroup is not None else frame_group(W * H, group)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    rs, rp, fc = _native(camera, params, config, histogram, True)
    fg.render(dv, rs, rp, fc, stream.cuda_stream)
    fg.finish(stream)
    if fg.rank != 0:
        return None
    pixels, small, _, _ = _lib.pinned.frame(H, W)
    fg.download(pixels, small, stream.cuda_stream)
    fg.release(stream.cuda_stream)
    hit_count = int(small[256])
    image_hist = small[:256]
    if int(small[258]) & 0xFFFFFFFF and params.max_steps <= 0:
        # a ray exhausted its own step budget: the exact frame budget, on rank 0
        d = render_detail(volume, camera, params, config, histogram, _checked=True)
        pixels, image_hist, hit_count = d.pixels, d.image_hist, d.hit_count
    total_ms = (time.perf_counter() - wall0) * 1000.0
    frame = Frame(pixels=pixels,
                  timing={"total_ms": total_ms, "march_ms": total_ms, "shade_ms": 0.0,
                          "device_ms": None, "ranks": fg.world},
                  filter_config=config, render_params=params, camera=camera,
                  volume_hash=volume.content_hash() if hasattr(volume, "content_hash") else "",
                  hit_count=hit_count)
    frame.image_hist = image_hist
    return frame
