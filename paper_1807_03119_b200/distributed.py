"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL).

Sort-first parallel rendering: every rank holds the full
volume replica and renders the 8x16-pixel tiles it owns (tile t belongs to
rank t % world, interleaved so early-terminating hit rays and long miss rays
balance); the partial frames (zero outside owned tiles) are summed onto rank
0 with one reduce, and the fused image histogram / hit count with one
all-reduce.  The Otsu histogram shards the volume into contiguous z-slabs:
each rank runs K1 on its slab and the 256 u64 bins are all-reduced, after
which every rank runs the K2 scan redundantly (identical T everywhere).

The communication helpers take torch tensors and work with any backend
(NCCL on the B200 box, gloo in the CPU tests).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

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
    """Sum 256-bin histograms across ranks (the 2 KiB NCCL all-reduce)."""
    import torch
    import torch.distributed as dist

    t = counts if isinstance(counts, torch.Tensor) else torch.as_tensor(
        np.asarray(counts, dtype=np.int64))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def reduce_frame(pixels, dst: int = 0, group=None):
    """Sum the ranks' partial frames (zero outside owned tiles) onto dst."""
    import torch.distributed as dist

    dist.reduce(pixels, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return pixels


def histogram_sharded(data: np.ndarray, group=None):
    """HistogramModel of a (nz, ny, nx) host volume, z-slab sharded (K1 + all-reduce + K2)."""
    import torch
    import torch.distributed as dist

    from . import _lib
    from .histogram import model_from_counts

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    z0, z1 = slab_bounds(data.shape[0], rank, world)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    slab = torch.from_numpy(np.array(data[z0:z1], copy=True).reshape(-1)).to(dev)
    counts = torch.zeros(256, dtype=torch.int64, device=dev)
    if slab.numel():
        _lib.call("vx_histogram_device", C.c_void_p(slab.data_ptr()), slab.numel(),
                  C.c_void_p(counts.data_ptr()), C.c_void_p(stream.cuda_stream))
    allreduce_counts(counts, group)
    return model_from_counts(counts.cpu().numpy())


def render_sharded(volume, camera, params, config, histogram=None, group=None):
    """Render one frame split over the group's GPUs; rank 0 gets the Frame."""
    import time

    import torch
    import torch.distributed as dist

    from . import _lib
    from .filters import native_config
    from .render import Frame, _check_render_args, native_params, ray_setup
    from .volume import device_volume

    wall0 = time.perf_counter()
    config = _check_render_args(config, histogram, None)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dv = device_volume(volume)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    W, H = params.width, params.height
    pixels = torch.zeros(H * W, dtype=torch.uint8, device=dev)
    small = torch.zeros(259, dtype=torch.int64, device=dev)
    out = _lib.vx_render_out()
    out.pixels = pixels.data_ptr()
    out.image_hist = small.data_ptr()
    out.hit_count = small.data_ptr() + 256 * 8
    out.trunc_flag = small.data_ptr() + 258 * 8
    rs = ray_setup(camera, W, H)
    rp = native_params(params)
    fc = native_config(config, histogram)
    part = _lib.vx_partition(rank, world)
    _lib.call("vx_render_device", dv.handle, C.byref(rs), C.byref(rp), C.byref(fc),
              C.byref(part), C.byref(out), C.c_void_p(stream.cuda_stream))
    reduce_frame(pixels, 0, group)
    dist.all_reduce(small, op=dist.ReduceOp.SUM, group=group)
    if int(small[258].item()) != 0 and params.max_steps <= 0:
        # a ray exhausted its own step budget: redo with the exact frame budget
        from .render import render_detail

        d = render_detail(volume, camera, params, config, histogram, partition=(rank, world))
        pixels.copy_(torch.from_numpy(d.pixels.reshape(-1)).to(dev))
        small[:256].copy_(torch.from_numpy(d.image_hist).to(dev))
        small[256] = d.hit_count
        small[258] = 0
        reduce_frame(pixels, 0, group)
        dist.all_reduce(small, op=dist.ReduceOp.SUM, group=group)
    if rank != 0:
        return None
    frame = Frame(pixels=pixels.cpu().numpy().reshape(H, W),
                  timing={"total_ms": (time.perf_counter() - wall0) * 1000.0,
                          "march_ms": 0.0, "shade_ms": 0.0},
                  filter_config=config, render_params=params, camera=camera,
                  volume_hash=volume.content_hash(), hit_count=int(small[256].item()))
    frame.image_hist = small[:256].cpu().numpy()
    return frame
