"""Pin the CPU oracle to the reference's golden vectors (CPU only).

The fixtures in tests/golden/ were produced by the live reference
(oracle/gen_golden.py); when /root/reference is importable the oracle is
additionally compared with it directly.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, golden

REF = Path("/root/reference/pkg/src")


def test_otsu_oracle_matches_reference_goldens(oracle):
    g = golden("otsu.npz")
    for counts, t in zip(g["counts"], g["threshold"]):
        assert oracle.otsu(counts) == t


def test_histogram_restatement(oracle):
    rs = np.random.default_rng(3)
    for n in (0, 1, 15, 16, 17, 1000, 65537):
        data = rs.integers(0, 256, n, dtype=np.uint8)
        assert np.array_equal(oracle.hist256(data), np.bincount(data, minlength=256))


def test_filter_oracle_matches_reference(oracle):
    g = golden("filters.npz")
    for vol, pts, kind, m, d, sc, bt in zip(g["volumes"], g["coords"], g["kinds"], g["kernel"],
                                            g["offset"], g["scalar"], g["batch"]):
        counts = np.bincount(vol.reshape(-1), minlength=256)
        h = oracle.histogram_model(counts)
        kw = dict(kind=str(kind), kernel_size=int(m), cluster_offset=int(d),
                  sigma_band=2.0 * h["global_sigma"], probabilities=h["probabilities"])
        got_b = oracle.filter_batch(vol, pts[:, 0], pts[:, 1], pts[:, 2], pairwise=False, **kw)
        assert np.array_equal(got_b, bt), kind
        got_s = np.array([oracle.filter_batch(vol, [p[0]], [p[1]], [p[2]], pairwise=True, **kw)[0]
                          for p in pts])
        assert np.array_equal(got_s, sc), kind


def test_ray_setup_oracle_bitwise(oracle):
    g = golden("shading.npz")
    for i in range(3):
        c = g[f"cam{i}"]
        pos, look, up, fov, w, h = c[0:3], c[3:6], c[6:9], c[9], int(c[10]), int(c[11])
        cam = oracle.cam_vector(tuple(pos), tuple(look), w, h, fov_y_deg=fov, up=tuple(up))
        d = oracle.ray_dirs(cam, w, h)
        assert np.array_equal(d, g[f"dirs{i}"])
        te, tx = oracle.ray_spans(pos, d, (9, 13, 64))
        assert np.array_equal(te, g[f"te{i}"]) and np.array_equal(tx, g[f"tx{i}"])
    for j in range(4):
        te, tx = oracle.ray_spans(g[f"par_o{j}"], g["par_dirs"], (5, 5, 5))
        np.testing.assert_array_equal(te, g[f"par_te{j}"])
        np.testing.assert_array_equal(tx, g[f"par_tx{j}"])


def test_sobel_phong_entropy_oracle(oracle):
    g = golden("shading.npz")
    pts = g["sobel_pts"]
    n = oracle.sobel_batch(g["sobel_vol"], pts[:, 0], pts[:, 1], pts[:, 2], g["sobel_fb"])
    assert np.array_equal(n, g["sobel_n"])
    px = oracle.phong_batch(g["phong_n"], g["phong_v"], g["phong_l"])
    # n.l in the reference is a BLAS dgemv: ulp-level order differences only
    assert (px != g["phong_px"]).sum() <= 2
    for i in range(4):
        assert oracle.image_entropy(g[f"img{i}"]) == float(g[f"img{i}_H"])


def test_u16_rescale_identity():
    g = golden("shading.npz")
    v = np.arange(65536, dtype=np.uint32)
    assert np.array_equal(((v + 128) // 257).astype(np.uint8), g["u16_rescale"])


@pytest.mark.parametrize("name", ["spot_64", "spot_128", "speckle_128", "latency_64"])
def test_frames_oracle_matches_reference(oracle, name):
    from oracle.rng_np import generate_phantom_np

    meta = json.loads((GOLDEN / "phantoms.json").read_text())[name]
    vol = generate_phantom_np(meta["spec"])
    assert hashlib.sha256(f"{vol.shape[2]}x{vol.shape[1]}x{vol.shape[0]}|".encode()
                          + vol.tobytes()).hexdigest() == meta["sha256"]
    g = golden("frames_small.npz")
    counts = oracle.hist256(vol)
    assert np.array_equal(counts, g[f"{name}__counts"])
    h = oracle.histogram_model(counts)
    assert h["otsu"] == int(g[f"{name}__otsu"])
    size = g[f"{name}__none__pixels"].shape[0]
    pos, look = oracle.orbit(vol.shape[::-1])
    cam = oracle.cam_vector(pos, look, size, size)
    for kind in ("none", "mean", "sigma", "entropy", "okada", "local-cluster"):
        r = oracle.render(vol, cam, size, size, kind=kind, threshold=float(h["otsu"]),
                          sigma_band=2.0 * h["global_sigma"], probabilities=h["probabilities"],
                          entropy_threshold=0.5 if kind == "entropy" else 2.0)
        key = f"{name}__{kind}"
        assert np.array_equal(r["pixels"], g[key + "__pixels"]), key
        assert r["hit_count"] == int(g[key + "__hits"]), key
        assert np.array_equal(r["hit_voxel"], g[key + "__voxel"].astype(np.int32)), key
        assert np.array_equal(r["hit_t"], g[key + "__t"]), key


def test_phantom_generators_match_reference_hashes(oracle):
    from oracle.rng_np import generate_phantom_np

    meta = json.loads((GOLDEN / "phantoms.json").read_text())
    for name in ("spot_64", "latency_64", "latency_128", "bench_128"):
        spec = meta[name]["spec"]
        for vol in (generate_phantom_np(spec), oracle.phantom(spec)):
            h = hashlib.sha256(f"{vol.shape[2]}x{vol.shape[1]}x{vol.shape[0]}|".encode()
                               + vol.tobytes()).hexdigest()
            assert h == meta[name]["sha256"], name


@pytest.mark.skipif(not (GOLDEN / "frames_c2.npz").exists(), reason="C2 fixture not frozen")
def test_c2_fixture_consistency(oracle):
    g = golden("frames_c2.npz")
    counts = g["counts"]
    assert oracle.otsu(counts) == int(g["otsu"])
    for kind in ("none", "mean", "sigma", "entropy", "okada", "local-cluster"):
        assert oracle.image_entropy(g[f"{kind}__pixels"]) == pytest.approx(float(g[f"{kind}__H"]),
                                                                          abs=1e-12)


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted (GPU box)")
def test_oracle_against_live_reference_random_cameras(oracle):
    sys.path.insert(0, str(REF))
    import voxray
    from voxray.render import Camera

    rs = np.random.default_rng(11)
    data = (rs.random((20, 24, 28)) < 0.05).astype(np.uint8) * 220 + rs.integers(0, 40, (20, 24, 28),
                                                                                   dtype=np.uint8)
    v = voxray.Volume(dims=(28, 24, 20), data=data)
    h = voxray.build_histogram(v)
    for trial in range(6):
        pos = tuple(float(x) for x in rs.uniform(-40, 70, 3))
        look = tuple(float(x) for x in rs.uniform(0, 20, 3))
        cam = Camera(position=pos, look_at=look, fov_y_deg=float(rs.uniform(20, 80)))
        step = [0.5, 0.37, 1.0, 2.5, 16.0, 0.5][trial]
        params = voxray.RenderParams(width=40, height=30, step_size=step)
        for kind in voxray.FilterKind:
            cfg = voxray.FilterConfig(kind=kind, threshold=float(rs.integers(0, 200)))
            f = voxray.render_frame(v, cam, params, cfg, h)
            cv = oracle.cam_vector(pos, look, 40, 30, fov_y_deg=cam.fov_y_deg)
            r = oracle.render(v.data, cv, 40, 30, kind=kind.value, threshold=cfg.threshold,
                              sigma_band=2.0 * h.global_sigma, probabilities=h.probabilities,
                              step=step)
            assert np.array_equal(r["pixels"], f.pixels), (trial, kind)
