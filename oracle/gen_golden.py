"""Freeze golden vectors from the LIVE reference (build container only).

    python -m oracle.gen_golden [--big]

Imports voxray from /root/reference/pkg/src (read-only, never copied) and
writes small fixtures under tests/golden/:

  otsu.npz          1000 random + adversarial histograms -> reference otsu()
  filters.npz       random 9^3 volumes x coords x kinds -> apply_filter(_batch)
  shading.npz       primary_ray_dirs / ray_box_spans / sobel_normal /
                    shade_phong / image_entropy reference outputs
  phantoms.json     sha256 of reference generate_phantom() volumes
  frames_small.npz  render_frame pixels + _march_batch hit voxels for the
                    committed phantoms (C1 spot_64 @256^2, spot_128,
                    speckle_128 @256^2, latency_64 @128^2), all six filters
  frames_c2.npz     (--big) C2/C3 insect_512 @1024^2, six filters: pixels,
                    hit-voxel digests, entropies, Otsu T

The GPU box has no /root/reference: tests read only these files.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _ref():
    sys.path.insert(0, str(REF_SRC))
    import voxray  # noqa: F401

    return voxray


def ref_hits(vx, volume, camera, params, config, hist):
    """Reference per-pixel hit voxels / t via its own _march_batch (render.py:467-476)."""
    from voxray import render as R
    from voxray.filters import apply_filter_batch

    config = config.resolve_threshold(hist)
    origin = np.asarray(camera.position, dtype=np.float64)
    dirs = R.primary_ray_dirs(camera, params.width, params.height)
    te, tx = R.ray_box_spans(origin, dirs, volume.dims)
    spans = np.where(tx >= te, tx - te, 0.0)
    max_steps = max(1, math.ceil(float(spans.max()) / params.step_size) + 1)

    def fn(xs, ys, zs):
        return apply_filter_batch(volume, xs, ys, zs, config, hist)

    hit, vox, ht, _ = R._march_batch(volume, origin, dirs, te, tx, float(config.threshold),
                                     params.step_size, max_steps, fn)
    vox = np.where(hit[:, None], vox, -1).astype(np.int32)
    return vox, ht.astype(np.float32)


def gen_otsu(vx):
    rs = np.random.default_rng(2024)
    cases = []
    for _ in range(1000):
        c = rs.integers(0, 1000, 256)
        c[rs.integers(0, 256, int(rs.integers(0, 250)))] = 0
        if c.sum() == 0:
            c[int(rs.integers(0, 256))] = 1
        cases.append(c)
    # adversarial: single bin, two-spike plateau, level-T class, big counts, spikes
    for b in (0, 1, 137, 255):
        c = np.zeros(256, dtype=np.int64); c[b] = 42; cases.append(c)
    c = np.zeros(256, dtype=np.int64); c[10] = 500; c[200] = 500; cases.append(c)
    c = np.zeros(256, dtype=np.int64); c[100] = 10; c[101] = 10; cases.append(c)
    big = rs.integers(0, 2 ** 36, 256); cases.append(big)          # ~2^44 voxels
    c = np.zeros(256, dtype=np.int64); c[0] = 2 ** 45; c[255] = 3; cases.append(c)
    c = np.full(256, 7, dtype=np.int64); cases.append(c)
    bg = rs.integers(0, 100, 256); bg[0] = 10 ** 9; cases.append(bg)  # CT background spike
    counts = np.stack([np.asarray(c, dtype=np.int64) for c in cases])
    t = np.array([vx.otsu([int(v) for v in c]) for c in counts], dtype=np.int32)
    np.savez_compressed(OUT / "otsu.npz", counts=counts, threshold=t)
    print("otsu", counts.shape)


def gen_filters(vx):
    from voxray.filters import apply_filter, apply_filter_batch

    rs = np.random.default_rng(77)
    vols, coords, kinds, ms, ds, scalar, batch = [], [], [], [], [], [], []
    variants = [(k, 3, 1) for k in vx.FilterKind] + [
        (vx.FilterKind.MEAN, 5, 1), (vx.FilterKind.SIGMA, 5, 1), (vx.FilterKind.ENTROPY, 5, 1),
        (vx.FilterKind.LOCAL_CLUSTER, 5, 2), (vx.FilterKind.LOCAL_CLUSTER, 3, 3)]
    for i in range(120):
        data = rs.integers(0, 256, (9, 9, 9), dtype=np.uint8)
        if i % 10 == 0:  # spiky / skewed volumes
            data = np.where(rs.random((9, 9, 9)) < 0.9, 0, 255).astype(np.uint8)
        v = vx.Volume(dims=(9, 9, 9), data=data)
        h = vx.build_histogram(v)
        pts = np.concatenate([rs.integers(2, 7, (3, 3)), rs.choice([0, 1, 7, 8], (3, 3)),
                              rs.integers(-3, 12, (2, 3))])
        for kind, m, d in variants:
            cfg = vx.FilterConfig(kind=kind, kernel_size=m, cluster_offset=d)
            b = apply_filter_batch(v, pts[:, 0], pts[:, 1], pts[:, 2], cfg, h)
            s = np.array([apply_filter(v, *map(int, p), cfg, h) for p in pts])
            vols.append(data); coords.append(pts); kinds.append(kind.value); ms.append(m)
            ds.append(d); scalar.append(s); batch.append(b)
    np.savez_compressed(OUT / "filters.npz", volumes=np.stack(vols), coords=np.stack(coords),
                        kinds=np.array(kinds), kernel=np.array(ms), offset=np.array(ds),
                        scalar=np.stack(scalar), batch=np.stack(batch))
    print("filters", len(kinds))


def gen_shading(vx):
    from voxray.metrics import image_entropy
    from voxray.render import (Camera, primary_ray_dirs, ray_box_spans, shade_phong_batch,
                               sobel_normal_batch)

    rs = np.random.default_rng(5)
    out = {}
    cams = [Camera(position=(50.0, -30.0, 20.0), look_at=(4.0, 4.0, 4.0)),
            Camera(position=(-7.5, 3.25, 100.0), look_at=(3.0, 2.0, 1.0), fov_y_deg=30.0),
            vx.orbit_camera(vx.Volume(dims=(64, 64, 64), data=np.zeros(64 ** 3, np.uint8)))]
    sizes = [(17, 11), (32, 32), (64, 48)]
    for i, (cam, (w, h)) in enumerate(zip(cams, sizes)):
        d = primary_ray_dirs(cam, w, h)
        te, tx = ray_box_spans(np.asarray(cam.position), d, (9, 13, 64))
        out[f"cam{i}"] = np.array([*cam.position, *cam.look_at, *cam.up, cam.fov_y_deg, w, h])
        out[f"dirs{i}"] = d
        out[f"te{i}"] = te
        out[f"tx{i}"] = tx
    # axis-parallel rays (parallel-slab branch) and an inside origin
    pd = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, -1.0], [0.6, 0.8, 0.0]])
    for j, o in enumerate([(-10.0, 2.0, 2.0), (2.0, 2.0, 2.0), (2.0, 9.0, 2.0), (-0.5, -0.5, 4.0)]):
        te, tx = ray_box_spans(np.asarray(o), pd, (5, 5, 5))
        out[f"par_o{j}"] = np.asarray(o)
        out[f"par_te{j}"] = te
        out[f"par_tx{j}"] = tx
    out["par_dirs"] = pd
    data = rs.integers(0, 256, (9, 9, 9), dtype=np.uint8)
    data[0:3, 0:3, 0:3] = 50  # flat corner -> fallback normal
    v = vx.Volume(dims=(9, 9, 9), data=data)
    pts = np.concatenate([rs.integers(0, 9, (200, 3)), [[1, 1, 1], [-1, 4, 4], [9, 9, 9]]])
    fb = rs.normal(size=(pts.shape[0], 3))
    fb /= np.linalg.norm(fb, axis=1, keepdims=True)
    out["sobel_vol"] = data
    out["sobel_pts"] = pts
    out["sobel_fb"] = fb
    out["sobel_n"] = sobel_normal_batch(v, pts[:, 0], pts[:, 1], pts[:, 2], fb)
    n = rs.normal(size=(5000, 3)); n /= np.linalg.norm(n, axis=1, keepdims=True)
    vv = rs.normal(size=(5000, 3)); vv /= np.linalg.norm(vv, axis=1, keepdims=True)
    light = np.array([1.0, -1.0, 1.5]); light /= np.linalg.norm(light)
    p = vx.RenderParams()
    out["phong_n"] = n
    out["phong_v"] = vv
    out["phong_l"] = light
    out["phong_px"] = shade_phong_batch(n, vv, light, p)
    imgs = [rs.integers(0, 256, (17, 23), dtype=np.uint8), np.full((8, 8), 77, np.uint8),
            np.repeat(np.arange(256, dtype=np.uint8), 4).reshape(32, 32),
            (rs.random((64, 64)) < 0.3).astype(np.uint8) * 200]
    for i, im in enumerate(imgs):
        out[f"img{i}"] = im
        out[f"img{i}_H"] = np.array(image_entropy(im))
    wide = np.arange(65536, dtype=np.float64)
    out["u16_rescale"] = np.floor(wide * 255.0 / 65535.0 + 0.5).astype(np.uint8)
    np.savez_compressed(OUT / "shading.npz", **out)
    print("shading", len(out))


SMALL = {
    "spot_64": ("spot_phantom_spec", 64, 256),
    "spot_128": ("spot_phantom_spec", 128, 256),
    "speckle_128": ("speckle_phantom_spec", 128, 256),
    "latency_64": ("latency_phantom_spec", 64, 128),
}


def _configs(vx):
    return [vx.FilterConfig(kind=vx.FilterKind.NONE), vx.FilterConfig(kind=vx.FilterKind.MEAN),
            vx.FilterConfig(kind=vx.FilterKind.SIGMA),
            vx.FilterConfig(kind=vx.FilterKind.ENTROPY, entropy_threshold=0.5),
            vx.FilterConfig(kind=vx.FilterKind.OKADA),
            vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER)]


def gen_frames(vx):
    import voxray.phantoms as P

    frames = {}
    hashes = {}
    for name, (fn, dims, size) in SMALL.items():
        spec = getattr(P, fn)(dims=dims)
        v = vx.generate_phantom(spec)
        hashes[name] = {"spec": spec.to_json(), "sha256": v.content_hash()}
        h = vx.build_histogram(v)
        cam = vx.orbit_camera(v)
        params = vx.RenderParams(width=size, height=size)
        frames[f"{name}__counts"] = h.counts
        frames[f"{name}__otsu"] = np.array(h.otsu_threshold)
        for cfg in _configs(vx):
            f = vx.render_frame(v, cam, params, cfg, h)
            vox, ht = ref_hits(vx, v, cam, params, cfg, h)
            key = f"{name}__{cfg.kind.value}"
            frames[key + "__pixels"] = f.pixels
            frames[key + "__hits"] = np.array(f.hit_count)
            frames[key + "__voxel"] = vox.astype(np.int16)
            frames[key + "__t"] = ht
            frames[key + "__H"] = np.array(vx.image_entropy(f.pixels))
        print("frames", name)
    np.savez_compressed(OUT / "frames_small.npz", **frames)
    return hashes


def gen_phantom_hashes(vx, hashes):
    import voxray.phantoms as P

    for name, fn, dims in (("latency_128", "latency_phantom_spec", 128),
                           ("bench_128", "bench_phantom_spec", 128)):
        spec = getattr(P, fn)(dims=dims)
        hashes[name] = {"spec": spec.to_json(), "sha256": vx.generate_phantom(spec).content_hash()}
    (OUT / "phantoms.json").write_text(json.dumps(hashes, indent=1, sort_keys=True) + "\n")


def insect_spec_ref(vx, n=512):
    """The C2 spec, built from reference primitives."""
    from voxray.phantoms import _blob_positions

    c = (n - 1) / 2
    shapes = []
    for dy, r, val in ((-150, 70, 190), (-30, 95, 170), (120, 110, 160)):
        shapes.append(vx.Shape(kind="sphere", center=(c, c + dy, c), radius=r, intensity=val))
        shapes.append(vx.Shape(kind="shell", center=(c, c + dy, c), radius=r, thickness=6,
                               intensity=230))
    for dy in (-70, -30, 10):
        for sx in (-1, 1):
            shapes.append(vx.Shape(kind="box", center=(c + sx * 150, c + dy, c - 60),
                                   extent=(200, 8, 8), intensity=210))
    for x, y, z in _blob_positions(n, 400, 220, 11):
        shapes.append(vx.Shape(kind="box", center=(float(x), float(y), float(z)),
                               extent=(3.0, 3.0, 1.0), intensity=200))
    return vx.PhantomSpec(dims=(n, n, n), shapes=tuple(shapes), noise_sigma=12.0,
                          spot_noise=vx.SpotNoise(density=2000.5 / n ** 3, intensity=255),
                          rng_seed=1807)


def gen_c2(vx):
    spec = insect_spec_ref(vx)
    t0 = time.time()
    v = vx.generate_phantom(spec)
    h = vx.build_histogram(v)
    print(f"insect_512 generated in {time.time() - t0:.1f}s T={h.otsu_threshold}")
    cam = vx.orbit_camera(v)
    params = vx.RenderParams(width=1024, height=1024)
    out = {"spec_json": np.array(json.dumps(spec.to_json())), "sha256": np.array(v.content_hash()),
           "counts": h.counts, "otsu": np.array(h.otsu_threshold)}
    for cfg in _configs(vx):
        t0 = time.time()
        f = vx.render_frame(v, cam, params, cfg, h)
        dt = time.time() - t0
        vox, ht = ref_hits(vx, v, cam, params, cfg, h)
        k = cfg.kind.value
        out[f"{k}__pixels"] = f.pixels
        out[f"{k}__hits"] = np.array(f.hit_count)
        out[f"{k}__voxel_sha"] = np.array(hashlib.sha256(vox.astype(np.int32).tobytes()).hexdigest())
        out[f"{k}__H"] = np.array(vx.image_entropy(f.pixels))
        out[f"{k}__ref_ms"] = np.array(dt * 1000.0)
        if k == "local-cluster":
            out[f"{k}__voxel"] = vox.astype(np.int16)
        print(f"c2 {k} {dt:.1f}s hits={f.hit_count} H={out[f'{k}__H']:.4f}")
    np.savez_compressed(OUT / "frames_c2.npz", **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also freeze the 512^3 C2/C3 frames")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    OUT.mkdir(parents=True, exist_ok=True)
    vx = _ref()
    only = set(args.only.split(",")) if args.only else None
    if not only or "otsu" in only:
        gen_otsu(vx)
    if not only or "filters" in only:
        gen_filters(vx)
    if not only or "shading" in only:
        gen_shading(vx)
    if not only or "frames" in only:
        hashes = gen_frames(vx)
        gen_phantom_hashes(vx, hashes)
    if args.big or (only and "c2" in only):
        gen_c2(vx)


if __name__ == "__main__":
    main()
