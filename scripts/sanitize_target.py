"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck; ONE tool per gpurun call -- see scripts/sanitize.sh).

Covers every kernel family with its concurrency machinery:
  K1+K2  hist_otsu_kernel incl. the last-block ticket and workspace reset,
         stand-alone K1 + K2, slab histogram of a replica;
  K3     volume build (cell / brick max, distance maps), u16 rescale, K7;
  K4     all six filters, whole and split rays (every frame scheduled by cost,
         1/16 of the tiles split in 8, 1/8 in 4, 1/8 in 2), the side-stream
         tile order, the warp-cooperative march (WarpScratch), the
         accepted-cell map build (K8) and the frame group's peer-slot path;
  K5     filter batch, Sobel / Phong batches, march_rays;
  K6     image entropy.
Pixels are checked against the oracle, so a clean sanitizer run is also a
correct one.  Exit code 0 = everything matched.
"""

from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> int:
    import paper_1807_03119_b200 as vx
    from oracle import oracle as orc
    from oracle.rng_np import generate_phantom_np
    from paper_1807_03119_b200 import _lib, phantoms
    from paper_1807_03119_b200.filters import native_config
    from paper_1807_03119_b200.render import native_params, ray_setup, render_detail
    from paper_1807_03119_b200.volume import device_volume

    _lib.require_device()
    spec = phantoms.spot_phantom_spec(48)
    data = generate_phantom_np(spec.to_json())
    vol = vx.Volume(dims=spec.dims, data=data)
    hist = vx.build_histogram(vol)
    assert np.array_equal(hist.counts, orc.hist256(data))
    assert vx.otsu(hist.counts) == orc.otsu(hist.counts)
    cam = vx.orbit_camera(vol)
    W, H = 72, 48
    params = vx.RenderParams(width=W, height=H)
    cv = orc.cam_vector(cam.position, cam.look_at, W, H)
    _lib.call("vx_set_schedule", 1, 0, 0, 1)  # order + split every frame
    bad = 0
    for kind in vx.FilterKind:
        cfg = vx.FilterConfig(kind=kind).resolve_threshold(hist)
        want = orc.render(data, cv, W, H, kind=kind.value, threshold=cfg.threshold,
                          sigma_band=2.0 * hist.global_sigma, probabilities=hist.probabilities,
                          entropy_threshold=cfg.entropy_threshold)
        for rep in range(3):  # raw map, accepted-cell map build, warm
            d = render_detail(vol, cam, params, cfg, hist, diagnostics=True)
            if not (np.array_equal(d.pixels, want["pixels"])
                    and np.array_equal(d.hit_voxel, want["hit_voxel"])):
                print(f"MISMATCH {kind.value} rep {rep}")
                bad += 1
        H_ = vx.image_entropy(d.pixels)
        if abs(H_ - orc.image_entropy(want["pixels"])) > 1e-12:
            print(f"ENTROPY MISMATCH {kind.value}")
            bad += 1
    _lib.call("vx_set_schedule", -1, -1, 16, 4)
    # K5 batches
    rs = np.random.default_rng(3)
    xs, ys, zs = (rs.integers(-2, 50, 200) for _ in range(3))
    cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER, threshold=60.0)
    got = vx.filters.apply_filter_batch(vol, xs, ys, zs, cfg, hist)
    ref = orc.filter_batch(data, xs, ys, zs, kind="local-cluster")
    bad += int(not np.array_equal(got, ref))
    fb = np.tile([0.0, 0.0, 1.0], (200, 1))
    bad += int(not np.array_equal(vx.render.sobel_normal_batch(vol, xs, ys, zs, fb),
                                  orc.sobel_batch(data, xs, ys, zs, fb)))
    # march_rays
    hit = vx.render.march_ray(vol, cam.position, np.subtract(cam.look_at, cam.position),
                              vx.FilterConfig(kind=vx.FilterKind.MEAN), hist)
    bad += int(hit is None)
    # frame group, in-process peer-slot path (two ranks, host-ordered)
    dv = device_volume(vol)
    cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER).resolve_threshold(hist)
    r_s, r_p, f_c = ray_setup(cam, W, H), native_params(params), native_config(cfg, hist)
    gs, bl = [], []
    for r in range(2):
        g = C.c_void_p()
        b = np.zeros(_lib.VX_GROUP_BLOB_BYTES, np.uint8)
        _lib.call("vx_group_create", r, 2, W * H, C.byref(g), _lib.ptr(b))
        gs.append(g)
        bl.append(b)
    allb = np.concatenate(bl)
    for g in gs:
        _lib.call("vx_group_connect", g, _lib.ptr(allb), _lib.VX_GROUP_SYNC_HOST)
    want = render_detail(vol, cam, params, cfg, hist).pixels.copy()
    for _ in range(3):
        for g in reversed(gs):
            _lib.call("vx_group_render", g, dv.handle, C.byref(r_s), C.byref(r_p), C.byref(f_c),
                      None, None)
        pix = np.zeros(W * H, np.uint8)
        cnt = np.zeros(259, np.uint64)
        _lib.call("vx_group_download", gs[0], _lib.ptr(pix), _lib.ptr(cnt), W * H, None)
        bad += int(not np.array_equal(pix.reshape(H, W), want))
        _lib.call("vx_group_release", gs[0], None)
    for g in gs:
        _lib.load().vx_group_destroy(g)
    # slab histogram of the replica (the multi-GPU z-slab shard)
    import torch

    counts = torch.zeros(256, dtype=torch.int64, device="cuda")
    for z0, z1 in ((0, 17), (17, 30), (30, 48)):
        _lib.call("vx_volume_histogram_slab", dv.handle, z0, z1, C.c_void_p(counts.data_ptr()),
                  None)
    torch.cuda.synchronize()
    bad += int(not np.array_equal(counts.cpu().numpy(), hist.counts))
    # u16 ingest path
    wide = (data.astype(np.uint16) * 257).astype("<u2")
    v16 = vx.Volume(dims=spec.dims, data=data)
    h = C.c_void_p()
    _lib.call("vx_volume_create_u16", _lib.ptr(np.ascontiguousarray(wide)), *spec.dims,
              C.byref(h))
    out = np.empty_like(data)
    _lib.call("vx_volume_read", h, _lib.ptr(out))
    bad += int(not np.array_equal(out, data))
    _lib.load().vx_volume_destroy(h)
    del v16
    print("sanitize target:", "OK" if bad == 0 else f"{bad} mismatches")
    return 0 if bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
