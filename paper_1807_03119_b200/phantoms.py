"""Phantom specs used by the tests, the bench and the comparison configs.

The committed demo phantoms mirror phantoms.py of the reference (same seeds
and layout constants, phantoms.py:35-167) so image-level expectations carry
over.  ``insect_phantom_spec`` is the BASELINE.json C2/C3 input (SURVEY.md
§8d): head / thorax / abdomen spheres with 6-voxel cuticle shells, six leg
boxes, slab speckle and spot noise, built only from reference primitives;
``scale`` scales it to 1024^3 / 2048^3 (the bench and C4 configs).
"""

from __future__ import annotations

import numpy as np

from . import rng
from .volume import PhantomSpec, Shape, SpotNoise

SPOT_PHANTOM_SEED = 20
SPECKLE_PHANTOM_SEED = 3
BENCH_PHANTOM_SEED = 5
LATENCY_PHANTOM_SEED = 5
INSECT_PHANTOM_SEED = 1807


def _exact_count_density(count: int, n_voxels: int) -> float:
    return (count + 0.5) / n_voxels


def spot_phantom_spec(dims: int = 128, seed: int = SPOT_PHANTOM_SEED) -> PhantomSpec:
    n = dims ** 3
    c = (dims - 1) / 2.0
    return PhantomSpec(
        dims=(dims, dims, dims),
        shapes=(Shape(kind="sphere", center=(c, c, c), radius=dims * 0.3125, intensity=200),),
        noise_sigma=10.0,
        spot_noise=SpotNoise(density=_exact_count_density(50, n), intensity=255),
        rng_seed=seed,
    )


_BLOB_TAG = 0x736C6162  # the reference's substream tag for texture centres
_BLOB_DRAWS = 10000     # draws before giving up (phantoms.py:49-68)


def blob_positions(dims: int, count: int, sphere_radius: float, seed: int):
    """Texture centres of the reference's phantoms (phantoms.py:49-68): draw i
    of the substream proposes the point ``6 + (draw words 3i..3i+2) mod
    (dims - 12)``; proposals within ``sphere_radius + 8`` of the volume centre,
    or within 10 voxels of an accepted centre, are dropped; the first
    ``count`` survivors in draw order are the centres.

    All proposals are formed at once; only the greedy spacing test runs per
    point.  Distances are compared squared (integer points, centre on the
    half-voxel grid: no rounding can flip a comparison)."""
    span = dims - 12
    words = rng.stream(rng.substream_seed(seed, _BLOB_TAG), 0, 3 * _BLOB_DRAWS)
    pts = 6 + (words.reshape(-1, 3) % np.uint64(span)).astype(np.int64)
    off = pts - (dims - 1) / 2.0
    pts = pts[(off * off).sum(axis=1) >= (sphere_radius + 8) ** 2]
    chosen = np.empty((0, 3), dtype=np.int64)
    for p in pts:
        if len(chosen) == count:
            break
        if len(chosen) and int(((chosen - p) ** 2).sum(axis=1).min()) < 100:
            continue
        chosen = np.vstack([chosen, p])
    return [tuple(int(v) for v in p) for p in chosen]


def speckle_phantom_spec(dims: int = 128, seed: int = SPECKLE_PHANTOM_SEED) -> PhantomSpec:
    n = dims ** 3
    c = (dims - 1) / 2.0
    radius = dims * 0.3125
    slabs = tuple(Shape(kind="box", center=(float(x), float(y), float(z)), extent=(3.0, 3.0, 1.0),
                        intensity=200)
                  for x, y, z in blob_positions(dims, 30, radius, seed))
    return PhantomSpec(
        dims=(dims, dims, dims),
        shapes=(Shape(kind="sphere", center=(c, c, c), radius=radius, intensity=200),) + slabs,
        noise_sigma=10.0,
        spot_noise=SpotNoise(density=_exact_count_density(60, n), intensity=255),
        rng_seed=seed,
    )


_CHECKER = tuple((dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)
                 if (dx + dy + dz) % 2 == 0)


def bench_phantom_spec(dims: int = 256, seed: int = BENCH_PHANTOM_SEED) -> PhantomSpec:
    c = (dims - 1) / 2.0
    radius = dims * 0.3125
    scale = (dims / 256) ** 3
    pos = blob_positions(dims, max(12, round(600 * scale)), radius, seed)
    n_checker = max(8, round(350 * scale))
    shapes = [Shape(kind="sphere", center=(c, c, c), radius=radius, intensity=200)]
    for x, y, z in pos[:n_checker]:
        shapes.extend(Shape(kind="box", center=(float(x + dx), float(y + dy), float(z + dz)),
                            extent=(0.8, 0.8, 0.8), intensity=255) for dx, dy, dz in _CHECKER)
    for x, y, z in pos[n_checker:]:
        shapes.append(Shape(kind="box", center=(float(x), float(y), float(z)),
                            extent=(3.0, 3.0, 1.0), intensity=200))
    return PhantomSpec(dims=(dims, dims, dims), shapes=tuple(shapes), noise_sigma=10.0,
                       rng_seed=seed)


def latency_phantom_spec(dims: int = 128, seed: int = LATENCY_PHANTOM_SEED) -> PhantomSpec:
    c = (dims - 1) / 2.0
    return PhantomSpec(
        dims=(dims, dims, dims),
        shapes=(Shape(kind="sphere", center=(c, c, c), radius=dims * 0.3125, intensity=200),),
        noise_sigma=3.0,
        rng_seed=seed,
    )


def insect_phantom_spec(dims: int = 512, seed: int = INSECT_PHANTOM_SEED) -> PhantomSpec:
    """CT-like insect phantom (SURVEY.md §8d C2 recipe, scaled by dims/512).

    Lengths (radii, shell thickness, leg boxes, offsets) scale with s =
    dims/512; the slab speckle count scales with s^2 and the spot count with
    s^3 (constant density), speckle extent stays 3x3x1 voxels.
    """
    s = dims / 512.0
    c = (dims - 1) / 2.0
    shapes = []
    for dy, r, val in ((-150, 70, 190), (-30, 95, 170), (120, 110, 160)):
        centre = (c, c + dy * s, c)
        shapes.append(Shape(kind="sphere", center=centre, radius=r * s, intensity=val))
        shapes.append(Shape(kind="shell", center=centre, radius=r * s, thickness=6 * s,
                            intensity=230))
    for dy in (-70, -30, 10):
        for sx in (-1, 1):
            shapes.append(Shape(kind="box", center=(c + sx * 150 * s, c + dy * s, c - 60 * s),
                                extent=(200 * s, 8 * s, 8 * s), intensity=210))
    n_slabs = int(round(400 * s * s))
    for x, y, z in blob_positions(dims, n_slabs, 220 * s, 11):
        shapes.append(Shape(kind="box", center=(float(x), float(y), float(z)),
                            extent=(3.0, 3.0, 1.0), intensity=200))
    n_spots = int(round(2000 * s ** 3))
    return PhantomSpec(dims=(dims, dims, dims), shapes=tuple(shapes), noise_sigma=12.0,
                       spot_noise=SpotNoise(density=(n_spots + 0.5) / dims ** 3, intensity=255),
                       rng_seed=seed)


CT_DITHER_SEED = 2048


def write_ct_u16(spec, path, seed: int = CT_DITHER_SEED, chunk: int = 1 << 28) -> "VolumeMeta":
    """The C4 input: a headerless 16-bit CT file of the
    phantom ``spec`` plus its ``.meta.json`` sidecar, such that load_raw's
    rescale (volume.py:148-150) returns the phantom's 8-bit voxels exactly:
    u16 = clamp(257*v8 + e, 0, 65535), dither e in [-128, 128]
    (vx_u16_dither_device).  Generated on the device (K7, then the dither
    kernel) and written chunk by chunk; an input generator, not a
    parity-bearing path."""
    import ctypes as C
    import json
    from pathlib import Path

    import numpy as np
    import torch

    from . import _lib
    from .volume import VolumeMeta, _phantom_args, meta_path_for

    _lib.require_device()
    nx, ny, nz = spec.dims
    n = nx * ny * nz
    table, n_shapes, nseed, spots, k = _phantom_args(spec)
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    v8 = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.call("vx_phantom_device", C.c_void_p(v8.data_ptr()), nx, ny, nz, _lib.ptr(table),
              n_shapes, float(spec.noise_sigma), nseed, _lib.ptr(spots), k,
              int(spec.spot_noise.intensity), sp)
    wide = torch.empty(min(chunk, n), dtype=torch.int16, device="cuda")
    host = torch.empty(min(chunk, n), dtype=torch.int16, pin_memory=True)
    path = Path(path)
    with open(path, "wb") as f:
        for i0 in range(0, n, chunk):
            m = min(chunk, n - i0)
            _lib.call("vx_u16_dither_device", C.c_void_p(v8.data_ptr() + i0), m, i0, seed,
                      C.c_void_p(wide.data_ptr()), sp)
            host[:m].copy_(wide[:m])
            torch.cuda.synchronize()
            f.write(memoryview(host[:m].numpy().view(np.uint8)))
    del v8, wide, host
    meta = VolumeMeta(dims=spec.dims, bit_depth=16, source="write_ct_u16")
    meta_path_for(path).write_text(json.dumps(meta.to_json()))
    return meta
