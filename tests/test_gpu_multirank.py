"""Multi-rank sort-first frames on the B200.

The frame group's data path -- every rank's K4 storing its tiles into rank
0's frame slot and adding its counters there with system-scope atomics -- is
exercised on one GPU: (1) in one process through the C-ABI (two group
handles, the in-process peer-pointer path), (2) as two processes through
``bench.py --gpus 2`` (CUDA-IPC mapped slot, host-ordered frames, the
functional mode of a one-GPU box).  Frames must be bit-identical to the
single-rank frame for any rank count, as the reference's worker bands are
(render.py:514-541, test_render.py:242-251).
"""

from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _native(vx, volume, hist, W, H, kind):
    from paper_1807_03119_b200.filters import native_config
    from paper_1807_03119_b200.render import native_params, ray_setup

    cam = vx.orbit_camera(volume)
    params = vx.RenderParams(width=W, height=H, background=3)
    cfg = vx.FilterConfig(kind=kind).resolve_threshold(hist)
    return cam, params, cfg, ray_setup(cam, W, H), native_params(params), native_config(cfg, hist)


@pytest.mark.parametrize("world", [2, 3])
def test_group_cabi_in_process(vx, small_sphere_volume, small_sphere_histogram, world):
    from paper_1807_03119_b200 import _lib
    from paper_1807_03119_b200.volume import device_volume

    lib = _lib.load()
    W, H = 97, 61
    cam, params, cfg, rs, rp, fc = _native(vx, small_sphere_volume, small_sphere_histogram, W, H,
                                           vx.FilterKind.LOCAL_CLUSTER)
    ref = vx.render_frame(small_sphere_volume, cam, params, cfg, small_sphere_histogram)
    dv = device_volume(small_sphere_volume)
    groups, blobs = [], []
    for r in range(world):
        g = C.c_void_p()
        b = np.zeros(_lib.VX_GROUP_BLOB_BYTES, np.uint8)
        _lib.call("vx_group_create", r, world, W * H, C.byref(g), _lib.ptr(b))
        groups.append(g)
        blobs.append(b)
    allb = np.concatenate(blobs)
    try:
        # one process, one GPU: the caller orders frames (host sync)
        for g in groups:
            _lib.call("vx_group_connect", g, _lib.ptr(allb), _lib.VX_GROUP_SYNC_AUTO)
            mode = C.c_int32(-9)
            _lib.call("vx_group_info", g, C.byref(mode), None)
            assert mode.value == _lib.VX_GROUP_SYNC_HOST
        for frame in range(3):  # slot reuse: frames 1, 2 (two slots), 3 (slot of frame 1)
            for r in reversed(range(world)):
                _lib.call("vx_group_render", groups[r], dv.handle, C.byref(rs), C.byref(rp),
                          C.byref(fc), None, None)
            pix = np.zeros(W * H, np.uint8)
            cnt = np.zeros(259, np.uint64)
            _lib.call("vx_group_download", groups[0], _lib.ptr(pix), _lib.ptr(cnt), W * H, None)
            assert np.array_equal(pix.reshape(H, W), ref.pixels), frame
            assert int(cnt[256]) == ref.hit_count
            assert np.array_equal(cnt[:256].astype(np.int64),
                                  np.bincount(ref.pixels.reshape(-1), minlength=256))
            _lib.call("vx_group_release", groups[0], None)
        # a third unreleased frame on rank 0 is refused (two slots)
        for _ in range(2):
            _lib.call("vx_group_render", groups[0], dv.handle, C.byref(rs), C.byref(rp),
                      C.byref(fc), None, None)
        with pytest.raises(_lib.NativeError, match="still held"):
            _lib.call("vx_group_render", groups[0], dv.handle, C.byref(rs), C.byref(rp),
                      C.byref(fc), None, None)
    finally:
        _lib.call("vx_synchronize")
        for g in groups:
            lib.vx_group_destroy(g)


def test_group_rejects_foreign_blobs():
    from paper_1807_03119_b200 import _lib

    lib = _lib.load()
    a, b = C.c_void_p(), C.c_void_p()
    ba = np.zeros(_lib.VX_GROUP_BLOB_BYTES, np.uint8)
    bb = np.zeros(_lib.VX_GROUP_BLOB_BYTES, np.uint8)
    _lib.call("vx_group_create", 0, 2, 1000, C.byref(a), _lib.ptr(ba))
    _lib.call("vx_group_create", 1, 2, 999, C.byref(b), _lib.ptr(bb))  # another frame size
    try:
        with pytest.raises(_lib.NativeError, match="does not belong"):
            _lib.call("vx_group_connect", a, _lib.ptr(np.concatenate([ba, bb])), -1)
    finally:
        lib.vx_group_destroy(a)
        lib.vx_group_destroy(b)


def _bench(*args, timeout=600):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=str(ROOT), env=env)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_two_ranks_match_one_rank():
    """bench.py --gpus 2 launches its two ranks itself; on a one-GPU box they
    share the GPU (IPC-mapped frame slot, host-ordered frames).  The frame is
    bit-identical to the single-rank frame."""
    common = ["--size", "256", "--image", "320", "--steps", "4", "--warmup", "3", "--no-cpu",
              "--orbit", "0", "--noskip-steps", "0", "--ncu", "off"]
    one = _bench("--gpus", "1", *common)
    two = _bench("--gpus", "2", *common)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["frame"]["sha256_16"] == one["frame"]["sha256_16"]
    assert two["frame"]["hits"] == one["frame"]["hits"]
    assert two["config"]["otsu_T"] == one["config"]["otsu_T"]
    assert two["e2e"]["value"] > 0 and two["value"] > 0


def test_group_device_flags_two_threads(vx, small_sphere_volume, small_sphere_histogram):
    """The device-sync protocol (stream-memop done / consumed flags, no host
    round trip per frame) with two ranks as two threads of one process on
    one GPU -- their flag waits are ordinary cross-stream waits of one
    context.  Rank 1 runs ahead freely (bounded by the two slots); every
    frame rank 0 downloads equals the single-rank frame."""
    import threading

    import torch

    from paper_1807_03119_b200 import _lib
    from paper_1807_03119_b200.volume import device_volume

    lib = _lib.load()
    assert lib.vx_group_probe_device_sync() == 0
    W, H = 88, 64
    dv = device_volume(small_sphere_volume)
    cams = [vx.orbit_camera(small_sphere_volume, azimuth_deg=20.0 * f) for f in range(8)]
    params = vx.RenderParams(width=W, height=H)
    cfg = vx.FilterConfig(kind=vx.FilterKind.MEAN).resolve_threshold(small_sphere_histogram)
    want = [vx.render_frame(small_sphere_volume, c, params, cfg, small_sphere_histogram).pixels.copy()
            for c in cams]
    from paper_1807_03119_b200.filters import native_config
    from paper_1807_03119_b200.render import native_params, ray_setup

    rp, fc = native_params(params), native_config(cfg, small_sphere_histogram)
    rss = [ray_setup(c, W, H) for c in cams]
    gs, bl = [], []
    for r in range(2):
        g = C.c_void_p()
        b = np.zeros(_lib.VX_GROUP_BLOB_BYTES, np.uint8)
        _lib.call("vx_group_create", r, 2, W * H, C.byref(g), _lib.ptr(b))
        gs.append(g)
        bl.append(b)
    allb = np.concatenate(bl)
    for g in gs:
        _lib.call("vx_group_connect", g, _lib.ptr(allb), _lib.VX_GROUP_SYNC_DEVICE)
    got, errors = [], []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            for f, rs in enumerate(rss):
                _lib.call("vx_group_render", gs[r], dv.handle, C.byref(rs), C.byref(rp),
                          C.byref(fc), C.c_void_p(st.cuda_stream), None)
                if r == 0:
                    pix = np.zeros(W * H, np.uint8)
                    _lib.call("vx_group_download", gs[0], _lib.ptr(pix), None, W * H,
                              C.c_void_p(st.cuda_stream))
                    got.append(pix.reshape(H, W))
                    _lib.call("vx_group_release", gs[0], C.c_void_p(st.cuda_stream))
            st.synchronize()
        except Exception as exc:  # surfaced below
            errors.append(exc)

    ts = [threading.Thread(target=rank, args=(r,)) for r in (1, 0)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    try:
        assert not errors, errors
        assert len(got) == len(want)
        for f, (a, b) in enumerate(zip(got, want)):
            assert np.array_equal(a, b), f
    finally:
        _lib.call("vx_synchronize")
        for g in gs:
            lib.vx_group_destroy(g)


def test_vx_init_multi_device_frames(vx, small_sphere_volume, small_sphere_histogram):
    """SURVEY §8b's vx_init + the multi-device volume/frame: the listed
    devices each hold a replica, a frame is split over them (here device 0
    listed three times: host-ordered, the same peer-slot data path) and
    equals the single-device frame; the slab-sharded histogram equals K1."""
    from paper_1807_03119_b200 import _lib
    from paper_1807_03119_b200.filters import native_config
    from paper_1807_03119_b200.render import native_params, ray_setup

    lib = _lib.load()
    ids = (C.c_int * 3)(0, 0, 0)
    _lib.call("vx_init", 3, ids)
    m = C.c_void_p()
    data = np.ascontiguousarray(small_sphere_volume.data)
    _lib.call("vx_multi_volume_create_u8", _lib.ptr(data), *small_sphere_volume.dims, C.byref(m))
    try:
        n, sync = C.c_int32(), C.c_int32()
        _lib.call("vx_multi_info", m, C.byref(n), C.byref(sync))
        assert n.value == 3 and sync.value == _lib.VX_GROUP_SYNC_HOST
        counts = np.zeros(256, np.uint64)
        _lib.call("vx_multi_histogram", m, _lib.ptr(counts))
        assert np.array_equal(counts.astype(np.int64), small_sphere_histogram.counts)
        for W, H, az in ((96, 72, 30.0), (130, 50, 200.0), (96, 72, 75.0)):
            cam = vx.orbit_camera(small_sphere_volume, azimuth_deg=az)
            params = vx.RenderParams(width=W, height=H)
            cfg = vx.FilterConfig(kind=vx.FilterKind.SIGMA).resolve_threshold(small_sphere_histogram)
            want = vx.render_frame(small_sphere_volume, cam, params, cfg, small_sphere_histogram)
            rs, rp = ray_setup(cam, W, H), native_params(params)
            fc = native_config(cfg, small_sphere_histogram)
            pix = np.zeros((H, W), np.uint8)
            hist = np.zeros(256, np.uint64)
            hits = np.zeros(1, np.uint64)
            out = _lib.vx_render_out()
            out.pixels, out.image_hist, out.hit_count = pix.ctypes.data, hist.ctypes.data, hits.ctypes.data
            _lib.call("vx_multi_render", m, C.byref(rs), C.byref(rp), C.byref(fc), C.byref(out))
            assert np.array_equal(pix, want.pixels), (W, H, az)
            assert int(hits[0]) == want.hit_count
            assert np.array_equal(hist.astype(np.int64),
                                  np.bincount(want.pixels.reshape(-1), minlength=256))
    finally:
        lib.vx_multi_destroy(m)
        _lib.call("vx_init", 1, (C.c_int * 1)(0))


def test_render_frame_devices_kwarg(vx, small_sphere_volume, small_sphere_histogram, monkeypatch):
    """render_frame(devices=...) (or VOXB200_DEVICES) splits the
    frame over those GPUs from this process; the pixels, hit count and fused
    histogram do not depend on it."""
    cam = vx.orbit_camera(small_sphere_volume, azimuth_deg=120.0)
    params = vx.RenderParams(width=200, height=120)
    cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER)
    one = vx.render_frame(small_sphere_volume, cam, params, cfg, small_sphere_histogram)
    two = vx.render_frame(small_sphere_volume, cam, params, cfg, small_sphere_histogram,
                          devices=[0, 0])
    assert np.array_equal(one.pixels, two.pixels) and one.hit_count == two.hit_count
    assert np.array_equal(one.image_hist, two.image_hist)
    from paper_1807_03119_b200 import render as vxr

    monkeypatch.setenv("VOXB200_DEVICES", "0,0,0")
    vxr._env_devices.clear()  # read once per process: re-read for the test
    try:
        three = vx.render_frame(small_sphere_volume, cam, params, cfg, small_sphere_histogram)
    finally:
        monkeypatch.delenv("VOXB200_DEVICES")
        vxr._env_devices.clear()
    assert np.array_equal(one.pixels, three.pixels)
    from paper_1807_03119_b200.render import multi_volume

    mv = multi_volume(small_sphere_volume, (0, 0, 0))
    assert np.array_equal(mv.histogram_counts(), small_sphere_histogram.counts)
