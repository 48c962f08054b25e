"""Acceptance criteria of the reference (tests/test_acceptance.py) on the B200
path, plus the metrics harness (tests/test_metrics.py)."""

from __future__ import annotations

import json
import statistics

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu


def _volume(vx, name):
    meta = json.loads((GOLDEN / "phantoms.json").read_text())[name]
    spec = vx.PhantomSpec.from_json(meta["spec"])
    v = vx.generate_phantom(spec)
    assert v.content_hash() == meta["sha256"]
    return spec, v


def test_spot_suppression(vx):
    from paper_1807_03119_b200.render import primary_ray_dirs

    spec, v = _volume(vx, "spot_128")
    h = vx.build_histogram(v)
    cam = vx.orbit_camera(v)
    params = vx.RenderParams(width=256, height=256)
    sphere = spec.shapes[0]
    dirs = primary_ray_dirs(cam, 256, 256)
    oc = np.asarray(cam.position) - np.asarray(sphere.center)
    b = dirs @ oc
    sil = ((b * b - (oc @ oc - sphere.radius ** 2)) >= 0).reshape(256, 256)
    dil = sil.copy()
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            dil |= np.roll(np.roll(sil, dy, 0), dx, 1)
    lc = vx.render_frame(v, cam, params, vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER), h)
    none = vx.render_frame(v, cam, params, vx.FilterConfig(kind=vx.FilterKind.NONE), h)
    assert int(((lc.pixels != 0) & ~dil).sum()) == 0
    assert int(((none.pixels != 0) & ~dil).sum()) >= 1
    assert h.otsu_threshold == 48


def test_entropy_ordering_matches_reference(vx):
    _, v = _volume(vx, "speckle_128")
    h = vx.build_histogram(v)
    cam = vx.orbit_camera(v)
    params = vx.RenderParams(width=256, height=256)
    g = golden("frames_small.npz")
    cfgs = {"none": vx.FilterConfig(kind=vx.FilterKind.NONE),
            "mean": vx.FilterConfig(kind=vx.FilterKind.MEAN),
            "sigma": vx.FilterConfig(kind=vx.FilterKind.SIGMA),
            "entropy": vx.FilterConfig(kind=vx.FilterKind.ENTROPY, entropy_threshold=0.5),
            "okada": vx.FilterConfig(kind=vx.FilterKind.OKADA),
            "local-cluster": vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER)}
    report, frames = vx.run_entropy_comparison(v, cam, params, list(cfgs.values()), h)
    H = {r["filter"]: r["entropy_bits"] for r in report.rows}
    for name in cfgs:
        assert H[name] == pytest.approx(float(g[f"speckle_128__{name}__H"]), abs=1e-12)
    assert H["local-cluster"] < H["mean"] <= H["none"]
    for name in ("mean", "sigma", "entropy", "okada"):
        assert H["local-cluster"] < H[name]


def test_timing_report(vx, small_sphere_volume, small_sphere_histogram):
    rep = vx.run_timing_benchmark(small_sphere_volume, vx.orbit_camera(small_sphere_volume),
                                  vx.RenderParams(width=24, height=24),
                                  [vx.FilterConfig(kind=vx.FilterKind.MEAN)], samples=4, warmup=1,
                                  histogram=small_sphere_histogram)
    t = rep.rows[0]["timing"]
    assert len(t["samples_ms"]) == 4
    assert t["median_ms"] == pytest.approx(statistics.median(t["samples_ms"]))
    assert len(t["device_samples_ms"]) == 4 and all(0 < d for d in t["device_samples_ms"])
    assert all(d <= w for d, w in zip(t["device_samples_ms"], t["samples_ms"]))
    assert rep.to_json()["machine"]
    with pytest.raises(ValueError):
        vx.run_entropy_comparison(small_sphere_volume, vx.orbit_camera(small_sphere_volume),
                                  vx.RenderParams(width=16, height=16), [])
    v = vx.Volume(dims=(8, 8, 8), data=np.zeros(512, np.uint8))
    rep, _ = vx.run_entropy_comparison(v, vx.orbit_camera(v), vx.RenderParams(width=16, height=16),
                                       [vx.FilterConfig(threshold=101)], vx.build_histogram(v))
    assert rep.rows[0]["entropy_bits"] == 0.0


def test_service_frame_message(vx, small_sphere_volume, small_sphere_histogram):
    """§8f row 1: the framed message equals the reference's pack_frame layout
    around the device frame (service.py:38-53, 168-183)."""
    from paper_1807_03119_b200.frames import FRAME_HEADER, pack_frame, render_message, unpack_header

    cam = vx.orbit_camera(small_sphere_volume)
    params = vx.RenderParams(width=48, height=40)
    cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER)
    msg = render_message(small_sphere_volume, cam, params, cfg, small_sphere_histogram, 7)
    ref = vx.render_frame(small_sphere_volume, cam, params, cfg, small_sphere_histogram)
    h = unpack_header(msg)
    assert h["magic"] == b"VXSF" and h["version"] == 1 and h["sequence"] == 7
    assert (h["width"], h["height"]) == (48, 40)
    assert h["digest"] == ref.filter_config.digest()
    body = bytes(msg[FRAME_HEADER.size:])
    assert body == ref.pixels.tobytes()
    want = pack_frame(7, 48, 40, h["render_ms"], ref.filter_config.digest(), ref.pixels.tobytes())
    assert bytes(msg) == want
