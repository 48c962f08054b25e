"""K4 ray caster parity on the B200 (mirrors tests/test_render.py and the
acceptance suite of the reference): FP64 ray setup bitwise, hit voxels and
pixels exactly equal to the reference / oracle on every frame."""

from __future__ import annotations

import hashlib
import json
import math

import numpy as np
import pytest

from conftest import GOLDEN, golden, vol_from

pytestmark = pytest.mark.gpu

KINDS = ("none", "mean", "sigma", "entropy", "okada", "local-cluster")


def cfg_for(vx, kind, **kw):
    k = vx.FilterKind.from_name(kind)
    if kind == "entropy" and "entropy_threshold" not in kw:
        kw["entropy_threshold"] = 0.5
    return vx.FilterConfig(kind=k, **kw)


# --- ray setup / shading bitwise ---------------------------------------------------


def test_primary_ray_dirs_and_spans_bitwise(vx):
    from paper_1807_03119_b200.render import primary_ray_dirs, ray_box_spans

    g = golden("shading.npz")
    for i in range(3):
        c = g[f"cam{i}"]
        cam = vx.Camera(position=tuple(c[0:3]), look_at=tuple(c[3:6]), up=tuple(c[6:9]),
                        fov_y_deg=float(c[9]))
        d = primary_ray_dirs(cam, int(c[10]), int(c[11]))
        assert np.array_equal(d, g[f"dirs{i}"])
        te, tx = ray_box_spans(np.asarray(cam.position), d, (9, 13, 64))
        assert np.array_equal(te, g[f"te{i}"]) and np.array_equal(tx, g[f"tx{i}"])
    for j in range(4):
        te, tx = ray_box_spans(g[f"par_o{j}"], g["par_dirs"], (5, 5, 5))
        np.testing.assert_array_equal(te, g[f"par_te{j}"])
        np.testing.assert_array_equal(tx, g[f"par_tx{j}"])


def test_sobel_and_phong_vs_reference(vx):
    from paper_1807_03119_b200.render import shade_phong_batch, sobel_normal_batch

    g = golden("shading.npz")
    v = vx.Volume(dims=(9, 9, 9), data=g["sobel_vol"])
    pts = g["sobel_pts"]
    n = sobel_normal_batch(v, pts[:, 0], pts[:, 1], pts[:, 2], g["sobel_fb"])
    assert np.array_equal(n, g["sobel_n"])
    px = shade_phong_batch(g["phong_n"], g["phong_v"], g["phong_l"], vx.RenderParams())
    assert (px != g["phong_px"]).sum() <= 2


def test_sobel_ramps_and_phong_goldens(vx):
    from paper_1807_03119_b200.render import shade_phong, sobel_normal

    n = 9
    idx = np.arange(n, dtype=np.uint8)
    for axis in range(3):
        shape = [1, 1, 1]
        shape[2 - axis] = n
        data = np.broadcast_to(idx.reshape(shape), (n, n, n)).copy()
        want = np.zeros(3)
        want[axis] = -1.0
        assert np.allclose(sobel_normal(vol_from(vx, data), 4, 4, 4), want, atol=1e-12)
        rev = vol_from(vx, data[::-1, ::-1, ::-1].copy())
        assert np.allclose(sobel_normal(rev, 4, 4, 4), -want, atol=1e-12)
    flat = vol_from(vx, np.full((9, 9, 9), 8, np.uint8))
    assert np.allclose(sobel_normal(flat, 4, 4, 4, fallback=(0.0, 1.0, 0.0)), (0, 1, 0))
    p = vx.RenderParams(ambient=0.1, diffuse=0.7, specular=0.2, shininess=16)
    assert shade_phong((0, 0, 1), (0, 0, 1), (0, 0, -1), p) == round(0.1 * 255)
    assert shade_phong((0, 0, 1), (0, 0, 1), (0, 0, 1),
                       vx.RenderParams(ambient=0.0, diffuse=1.0, specular=0.0)) == 255


# --- march_ray known answers (test_render.py TestMarchRay) ---------------------------------


def test_march_ray_known_answers(vx, spot_volume):
    from paper_1807_03119_b200.render import march_ray

    v = vol_from(vx, np.zeros((9, 9, 9), np.uint8))
    assert march_ray(v, (-5, 4, 4), (1, 0, 0), vx.FilterConfig(kind=vx.FilterKind.MEAN,
                                                                threshold=101)) is None
    data = np.zeros((9, 9, 9), np.uint8)
    data[:, :, 5:] = 200
    slab = vol_from(vx, data)
    for kind in vx.FilterKind:
        h = vx.build_histogram(slab)
        hit = march_ray(slab, (-5, 4, 4), (1, 0, 0), vx.FilterConfig(kind=kind, threshold=101), h)
        assert hit is not None and hit.voxel[0] == 5 and hit.value >= 101, kind
    h = vx.build_histogram(spot_volume)
    lc = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER, threshold=101)
    none = vx.FilterConfig(kind=vx.FilterKind.NONE, threshold=101)
    assert march_ray(spot_volume, (-5.0, 4.0, 4.0), (1.0, 0.0, 0.0), lc, h) is None
    hit = march_ray(spot_volume, (-5.0, 4.0, 4.0), (1.0, 0.0, 0.0), none, h)
    assert hit is not None and hit.voxel == (4, 4, 4)
    data = np.array(spot_volume.data, copy=True)
    data[:, :, 7:] = 200
    v2 = vol_from(vx, data)
    hit = march_ray(v2, (-5.0, 4.0, 4.0), (1.0, 0.0, 0.0), lc, vx.build_histogram(v2))
    assert hit is not None and hit.voxel[0] == 7
    data = np.zeros((9, 9, 9), np.uint8)
    data[:, :, 6:] = 200
    v3 = vol_from(vx, data)
    mcfg = vx.FilterConfig(kind=vx.FilterKind.MEAN, threshold=101)
    hit = march_ray(v3, (2.0, 4.0, 4.0), (1.0, 0.0, 0.0), mcfg)
    assert hit is not None and hit.voxel[0] == 6
    assert march_ray(v3, (2.0, 4.0, 4.0), (-1.0, 0.0, 0.0), mcfg) is None
    hit = march_ray(vol_from(vx, np.zeros((9, 9, 9), np.uint8)), (-5.0, 4.0, 4.0), (1.0, 0.0, 0.0),
                    vx.FilterConfig(kind=vx.FilterKind.NONE, threshold=0))
    assert hit is not None and hit.voxel[0] == 0


# --- frames vs the reference's frozen frames -------------------------------------------------


@pytest.mark.parametrize("name", ["spot_64", "spot_128", "speckle_128", "latency_64"])
@pytest.mark.parametrize("skip", [True, False])
def test_frames_match_reference(vx, name, skip):
    from oracle.rng_np import generate_phantom_np
    from paper_1807_03119_b200.render import render_detail

    meta = json.loads((GOLDEN / "phantoms.json").read_text())[name]
    spec = vx.PhantomSpec.from_json(meta["spec"])
    v = vx.Volume(dims=spec.dims, data=generate_phantom_np(meta["spec"]))
    g = golden("frames_small.npz")
    h = vx.build_histogram(v)
    assert np.array_equal(h.counts, g[f"{name}__counts"])
    assert h.otsu_threshold == int(g[f"{name}__otsu"])
    size = g[f"{name}__none__pixels"].shape[0]
    cam = vx.orbit_camera(v)
    params = vx.RenderParams(width=size, height=size)
    # with skip, the second frame of a filter setting marches on its
    # accepted-cell map (vx_render.cu get_accept_map): both must match
    for kind, rep in [(k, r) for k in KINDS for r in range(2 if skip else 1)]:
        key = f"{name}__{kind}"
        d = render_detail(v, cam, params, cfg_for(vx, kind), h, diagnostics=True, skip=skip)
        assert np.array_equal(d.hit_voxel, g[key + "__voxel"].astype(np.int32)), key
        assert np.array_equal(d.pixels, g[key + "__pixels"]), key
        hit = d.hit_voxel[:, 0] >= 0
        assert np.array_equal(d.hit_t[hit], g[key + "__t"][hit]), key
        assert d.hit_count == int(g[key + "__hits"]), key
        assert np.array_equal(d.image_hist, np.bincount(d.pixels.reshape(-1), minlength=256))


def test_render_frame_api(vx, small_sphere_volume, small_sphere_histogram):
    from paper_1807_03119_b200.render import RenderError

    v = vol_from(vx, np.zeros((16, 16, 16), np.uint8))
    frame = vx.render_frame(v, vx.orbit_camera(v), vx.RenderParams(width=32, height=32,
                                                                   background=13),
                            vx.FilterConfig(threshold=101), vx.build_histogram(v))
    assert (frame.pixels == 13).all() and frame.hit_count == 0
    params = vx.RenderParams(width=64, height=64)
    cam = vx.orbit_camera(small_sphere_volume)
    f = vx.render_frame(small_sphere_volume, cam, params, vx.FilterConfig(kind=vx.FilterKind.MEAN),
                        small_sphere_histogram)
    assert f.hit_count > 200 and f.pixels.shape == (64, 64) and f.timing["total_ms"] > 0
    assert f.timing["device_ms"] is None
    from paper_1807_03119_b200.render import frame_timing

    with frame_timing():
        f = vx.render_frame(small_sphere_volume, vx.orbit_camera(small_sphere_volume), params,
                            vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER),
                            small_sphere_histogram)
    assert 0 < f.timing["device_ms"] == f.timing["march_ms"] <= f.timing["total_ms"]
    frames = [vx.render_frame(small_sphere_volume, cam, params,
                              vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER),
                              small_sphere_histogram, workers=w) for w in (1, 2, 5)]
    assert all((fr.pixels == frames[0].pixels).all() for fr in frames)
    meta = vx.render_frame(small_sphere_volume, cam, params,
                           vx.FilterConfig(kind=vx.FilterKind.OKADA),
                           small_sphere_histogram).meta_json()
    assert meta["filter_config"]["threshold"] == float(small_sphere_histogram.otsu_threshold)
    assert meta["volume_hash"] == small_sphere_volume.content_hash()
    with pytest.raises(RenderError):
        vx.render_frame(small_sphere_volume, cam, params, vx.FilterConfig(), small_sphere_histogram,
                        filter_fn=lambda x, y, z: x)
    with pytest.raises(RenderError, match="histogram"):
        vx.render_frame(small_sphere_volume, cam, params,
                        vx.FilterConfig(kind=vx.FilterKind.SIGMA, threshold=50.0))


# --- randomised parity vs the oracle -------------------------------------------------------


def test_random_cameras_steps_thresholds_vs_oracle(vx, oracle):
    from paper_1807_03119_b200.render import render_detail

    rs = np.random.default_rng(2)
    data = (rs.random((40, 48, 56)) < 0.02).astype(np.uint8) * 230 + rs.integers(
        0, 60, (40, 48, 56), dtype=np.uint8)
    data[10:30, 12:36, 14:42] = np.maximum(data[10:30, 12:36, 14:42], 150)
    v = vol_from(vx, data)
    h = vx.build_histogram(v)
    steps = [0.5, 0.37, 1.0, 2.5, 16.0, 0.5, 0.25, 3.0]
    for trial, step in enumerate(steps):
        pos = tuple(float(x) for x in rs.uniform(-80, 140, 3))
        look = tuple(float(x) for x in rs.uniform(5, 40, 3))
        fov = float(rs.uniform(15, 90))
        cam = vx.Camera(position=pos, look_at=look, fov_y_deg=fov)
        w, hh = int(rs.integers(20, 70)), int(rs.integers(20, 70))
        params = vx.RenderParams(width=w, height=hh, step_size=step,
                                 max_steps=int(rs.integers(5, 200)) if trial == 5 else 0)
        cv = oracle.cam_vector(pos, look, w, hh, fov_y_deg=fov)
        for kind in KINDS:
            T = float(rs.choice([0.0, 40.5, 67.0, 149.0, 231.0, 300.0]))
            cfg = cfg_for(vx, kind, threshold=T)
            want = oracle.render(data, cv, w, hh, kind=kind, threshold=T,
                                 sigma_band=2.0 * h.global_sigma, probabilities=h.probabilities,
                                 entropy_threshold=cfg.entropy_threshold, step=step,
                                 max_steps=params.max_steps)
            for skip in (True, True, False):  # raw map, accepted-cell map, no skip
                d = render_detail(v, cam, params, cfg, h, diagnostics=True, skip=skip)
                assert np.array_equal(d.hit_voxel, want["hit_voxel"]), (trial, kind, T, skip)
                assert np.array_equal(d.pixels, want["pixels"]), (trial, kind, T, skip)
                hit = want["hit_voxel"][:, 0] >= 0
                np.testing.assert_allclose(d.intensity[hit], want["intensity"][hit], atol=1e-12)


def test_cluster_and_mean_kernel_sizes_vs_oracle(vx, oracle):
    """Local cluster at M = 3/5/7 and d = 1-4 (filters.py:154-184), box mean
    and sigma at M = 3/5/7 (filters.py:173-195): the march's first-candidate evaluation
    splits the taps over the warp when few lanes need it, and must give the
    oracle's hit voxels and pixels."""
    from paper_1807_03119_b200.render import render_detail

    rs = np.random.default_rng(11)
    data = rs.integers(0, 90, (36, 40, 44), dtype=np.uint8)
    data[(rs.random(data.shape) < 0.01)] = 240
    data[8:28, 10:30, 12:34] = np.maximum(data[8:28, 10:30, 12:34], 170)
    v = vol_from(vx, data)
    h = vx.build_histogram(v)
    for trial, (m, d) in enumerate([(3, 1), (5, 1), (5, 2), (7, 3), (3, 4)]):
        pos = tuple(float(x) for x in rs.uniform(-60, 110, 3))
        cam = vx.Camera(position=pos, look_at=(22.0, 20.0, 18.0), fov_y_deg=40.0)
        w, hh = 48, 40
        params = vx.RenderParams(width=w, height=hh, step_size=0.5)
        cv = oracle.cam_vector(pos, (22.0, 20.0, 18.0), w, hh, fov_y_deg=40.0)
        for kind, T in (("local-cluster", 100.0), ("local-cluster", 150.0), ("mean", 120.0),
                        ("sigma", 120.0)):
            cfg = vx.FilterConfig(kind=vx.FilterKind.from_name(kind), threshold=T, kernel_size=m,
                                  cluster_offset=d)
            want = oracle.render(data, cv, w, hh, kind=kind, threshold=T, kernel_size=m,
                                 cluster_offset=d, sigma_band=2.0 * h.global_sigma)
            for skip in (True, True, False):
                got = render_detail(v, cam, params, cfg, h, diagnostics=True, skip=skip)
                assert np.array_equal(got.hit_voxel, want["hit_voxel"]), (trial, kind, m, d, T, skip)
                assert np.array_equal(got.pixels, want["pixels"]), (trial, kind, m, d, T, skip)


def test_partitions_sum_to_full_frame(vx, small_sphere_volume, small_sphere_histogram):
    from paper_1807_03119_b200.render import render_detail

    cam = vx.orbit_camera(small_sphere_volume)
    params = vx.RenderParams(width=61, height=45)
    cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER)
    full = render_detail(small_sphere_volume, cam, params, cfg, small_sphere_histogram)
    for world in (2, 3, 4, 8):
        acc = np.zeros_like(full.pixels, dtype=np.int64)
        owned = np.zeros_like(full.pixels, dtype=np.int64)
        hits = 0
        for r in range(world):
            d = render_detail(small_sphere_volume, cam, params, cfg, small_sphere_histogram,
                              partition=(r, world))
            acc += d.pixels
            hits += d.hit_count
        assert np.array_equal(acc, full.pixels) and hits == full.hit_count, world


# --- C2 / C3 (512^3 insect, 1024^2) against the frozen reference frames --------------------


@pytest.mark.skipif(not (GOLDEN / "frames_c2.npz").exists(), reason="C2 fixture not frozen")
def test_c2_c3_frames_match_reference(vx):
    from paper_1807_03119_b200 import phantoms
    from paper_1807_03119_b200.metrics import entropy_from_counts
    from paper_1807_03119_b200.render import render_detail
    from paper_1807_03119_b200.volume import generate_phantom_device

    g = golden("frames_c2.npz")
    spec = phantoms.insect_phantom_spec(512)
    dev = generate_phantom_device(spec)
    data = dev.read()
    v = vx.Volume(dims=spec.dims, data=data)
    object.__setattr__(v, "_vx_device", dev)
    if v.content_hash() != str(g["sha256"]):
        pytest.fail("device phantom differs from the reference phantom bytes")
    h = vx.build_histogram(v)
    assert np.array_equal(h.counts, g["counts"]) and h.otsu_threshold == int(g["otsu"])
    cam = vx.orbit_camera(v)
    params = vx.RenderParams(width=1024, height=1024)
    for kind, rep in [(k, r) for k in KINDS for r in range(2)]:  # raw map, accepted-cell map
        d = render_detail(v, cam, params, cfg_for(vx, kind), h, diagnostics=True)
        assert hashlib.sha256(d.hit_voxel.tobytes()).hexdigest() == str(g[f"{kind}__voxel_sha"]), kind
        assert np.array_equal(d.pixels, g[f"{kind}__pixels"]), kind
        assert d.hit_count == int(g[f"{kind}__hits"])
        H = entropy_from_counts(d.image_hist, 1024 * 1024)
        assert abs(H - float(g[f"{kind}__H"])) <= 1e-12
        assert abs(vx.image_entropy(d.pixels) - float(g[f"{kind}__H"])) <= 1e-3


def test_partition_matches_owned_mask(vx, small_sphere_volume, small_sphere_histogram):
    from paper_1807_03119_b200.distributed import owned_pixel_mask
    from paper_1807_03119_b200.render import render_detail

    cam = vx.orbit_camera(small_sphere_volume)
    params = vx.RenderParams(width=70, height=50, background=7)
    cfg = vx.FilterConfig(kind=vx.FilterKind.MEAN)
    full = render_detail(small_sphere_volume, cam, params, cfg, small_sphere_histogram).pixels
    for world in (2, 3):
        for r in range(world):
            d = render_detail(small_sphere_volume, cam, params, cfg, small_sphere_histogram,
                              partition=(r, world))
            m = owned_pixel_mask(70, 50, r, world)
            assert np.array_equal(d.pixels, np.where(m, full, 0))


def test_sharded_api_single_rank_nccl(vx, small_sphere_volume, small_sphere_histogram):
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_1807_03119_b200.distributed import histogram_sharded, render_sharded

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        h = histogram_sharded(small_sphere_volume)
        assert np.array_equal(h.counts, small_sphere_histogram.counts)
        assert h.otsu_threshold == small_sphere_histogram.otsu_threshold
        cam = vx.orbit_camera(small_sphere_volume)
        params = vx.RenderParams(width=64, height=40)
        cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER)
        f = render_sharded(small_sphere_volume, cam, params, cfg, h)
        ref = vx.render_frame(small_sphere_volume, cam, params, cfg, h)
        assert np.array_equal(f.pixels, ref.pixels) and f.hit_count == ref.hit_count
        assert np.array_equal(f.image_hist, np.bincount(ref.pixels.reshape(-1), minlength=256))
    finally:
        dist.destroy_process_group()


@pytest.fixture
def split_everything():
    """Schedule every frame's tiles by cost and split the rays of 1/16 of the
    tiles in 8 segments, 1/8 in 4 and 1/8 in 2, down to one
    chunk per segment (production only splits the heaviest tiles of big
    frames, and only rays of >= 8 chunks per segment); restored afterwards."""
    from paper_1807_03119_b200 import _lib

    _lib.call("vx_set_schedule", 1, 0, 0, 1)
    yield
    _lib.call("vx_set_schedule", -1, -1, 16, 4)


def test_split_rays_and_tile_order_match_oracle(vx, oracle, split_everything):
    """Frames 2+ of a setting run with the cost-ordered tiles and 8/4/2-segment
    rays (segment s starts from the exact chunk base of its first sample):
    hit voxels and pixels equal the oracle's, for every filter and steps that
    exercise the chunk rule."""
    from paper_1807_03119_b200.render import render_detail

    rs = np.random.default_rng(11)
    data = (rs.random((48, 40, 56)) < 0.03).astype(np.uint8) * 230 + rs.integers(
        0, 60, (48, 40, 56), dtype=np.uint8)
    data[8:30, 10:30, 12:40] = np.maximum(data[8:30, 10:30, 12:40], 160)
    v = vol_from(vx, data)
    h = vx.build_histogram(v)
    for trial, step in enumerate([0.5, 0.37, 1.0, 2.5]):
        pos = tuple(float(x) for x in rs.uniform(-90, 150, 3))
        look = tuple(float(x) for x in rs.uniform(5, 40, 3))
        cam = vx.Camera(position=pos, look_at=look, fov_y_deg=float(rs.uniform(20, 70)))
        w, hh = int(rs.integers(40, 90)), int(rs.integers(40, 90))
        params = vx.RenderParams(width=w, height=hh, step_size=step)
        cv = oracle.cam_vector(pos, look, w, hh, fov_y_deg=cam.fov_y_deg)
        for kind in KINDS:
            T = float(rs.choice([40.5, 67.0, 149.0]))
            cfg = cfg_for(vx, kind, threshold=T)
            want = oracle.render(data, cv, w, hh, kind=kind, threshold=T,
                                 sigma_band=2.0 * h.global_sigma, probabilities=h.probabilities,
                                 entropy_threshold=cfg.entropy_threshold, step=step)
            for rep in range(3):
                d = render_detail(v, cam, params, cfg, h, diagnostics=rep == 2)
                assert np.array_equal(d.pixels, want["pixels"]), (trial, kind, T, rep)
                if rep == 2:
                    assert np.array_equal(d.hit_voxel, want["hit_voxel"]), (trial, kind, T)


def test_concurrent_render_frame_threads(vx):
    """The reference service renders from executor threads on one shared
    volume (service.py:234-236): four threads, each with its own cameras and
    filter settings, give the same frames as a single-threaded render."""
    import threading

    from paper_1807_03119_b200 import phantoms
    from oracle.rng_np import generate_phantom_np

    spec = phantoms.spot_phantom_spec(64)
    v = vx.Volume(dims=spec.dims, data=generate_phantom_np(spec.to_json()))
    h = vx.build_histogram(v)
    kinds = [vx.FilterKind.LOCAL_CLUSTER, vx.FilterKind.MEAN, vx.FilterKind.NONE,
             vx.FilterKind.ENTROPY]
    jobs = []
    for w in range(4):
        for r in range(3):
            cam = vx.orbit_camera(v, azimuth_deg=30.0 * w + 11.0 * r, elevation_deg=10.0 + 7 * r)
            cfg = vx.FilterConfig(kind=kinds[(w + r) % 4])
            jobs.append((w, cam, cfg))
    # 320x300 = 760 tiles: above the scheduler's threshold, so each thread's
    # cost-ordered tiles, split rays and side-stream ordering are exercised
    params = vx.RenderParams(width=320, height=300)
    want = {i: vx.render_frame(v, cam, params, cfg, h).pixels.copy()
            for i, (_, cam, cfg) in enumerate(jobs)}
    got, errors = {}, []

    def worker(w):
        try:
            for rep in range(4):
                for i, (ww, cam, cfg) in enumerate(jobs):
                    if ww == w:
                        got[(i, rep)] = vx.render_frame(v, cam, params, cfg, h).pixels.copy()
        except Exception as exc:  # surfaced below
            errors.append(exc)

    ts = [threading.Thread(target=worker, args=(w,)) for w in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for (i, rep), px in got.items():
        assert np.array_equal(px, want[i]), (i, rep)
    assert len(got) == len(jobs) * 4


def test_map_cache_eviction_stress_threads(vx):
    """Six threads x six filter settings on one shared volume: more distinct
    thresholds (candidate distance maps) and filter settings (accepted-cell
    maps) than the volume's 4 + 4 cached map slots, so maps are evicted and
    rebuilt while other threads' frames are in flight.  A slot is pinned
    from lookup to K4 launch and rebuilt only after its readers (per-stream
    use events), so every frame equals its single-threaded render."""
    import threading

    from oracle.rng_np import generate_phantom_np
    from paper_1807_03119_b200 import phantoms

    spec = phantoms.spot_phantom_spec(64)
    v = vx.Volume(dims=spec.dims, data=generate_phantom_np(spec.to_json()))
    h = vx.build_histogram(v)
    kinds = [vx.FilterKind.LOCAL_CLUSTER, vx.FilterKind.MEAN, vx.FilterKind.SIGMA]
    settings = [vx.FilterConfig(kind=kinds[i % 3], threshold=float(t))
                for i, t in enumerate((30, 46, 61, 80, 101, 125))]
    params = vx.RenderParams(width=320, height=300)
    cams = [vx.orbit_camera(v, azimuth_deg=17.0 * w, elevation_deg=5.0 + 6 * w) for w in range(6)]
    want = {(w, s): vx.render_frame(v, cams[w], params, settings[s], h).pixels.copy()
            for w in range(6) for s in range(6)}
    bad, errors = [], []

    def worker(w):
        try:
            order = np.random.default_rng(w).permutation(6 * 5) % 6
            for s in order:
                px = vx.render_frame(v, cams[w], params, settings[s], h).pixels
                if not np.array_equal(px, want[(w, s)]):
                    bad.append((w, int(s)))
        except Exception as exc:  # surfaced below
            errors.append(exc)

    ts = [threading.Thread(target=worker, args=(w,)) for w in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    assert not bad, bad


def test_orbiting_camera_frames_match_oracle(vx, oracle):
    """A camera moving 3 degrees per frame: the tile order and split rays come
    from the previous frame's costs (a moving camera's schedule); whatever
    the schedule, every frame equals the oracle's."""
    from oracle.rng_np import generate_phantom_np
    from paper_1807_03119_b200 import phantoms
    from paper_1807_03119_b200.render import render_detail

    spec = phantoms.spot_phantom_spec(64)
    data = generate_phantom_np(spec.to_json())
    v = vx.Volume(dims=spec.dims, data=data)
    h = vx.build_histogram(v)
    W, H = 320, 304  # 760 tiles: above the scheduler's threshold
    params = vx.RenderParams(width=W, height=H)
    cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER).resolve_threshold(h)
    for k in range(8):
        cam = vx.orbit_camera(v, azimuth_deg=20.0 + 3.0 * k, elevation_deg=15.0 + k)
        d = render_detail(v, cam, params, cfg, h, diagnostics=True)
        want = oracle.render(data, oracle.cam_vector(cam.position, cam.look_at, W, H), W, H,
                             kind="local-cluster", threshold=cfg.threshold)
        assert np.array_equal(d.hit_voxel, want["hit_voxel"]), k
        assert np.array_equal(d.pixels, want["pixels"]), k
