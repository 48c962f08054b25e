"""Host-side logic of the drop-in (CPU only): validation errors and messages,
JSON round trips, offset tables, phantom specs, the native struct packing."""

from __future__ import annotations

import json
import math

import numpy as np
import pytest

from conftest import GOLDEN, golden


def test_filter_config_validation(vx):
    from paper_1807_03119_b200.filters import FilterError

    with pytest.raises(FilterError):
        vx.FilterConfig(kernel_size=4)
    with pytest.raises(FilterError):
        vx.FilterConfig(kernel_size=1)
    with pytest.raises(FilterError):
        vx.FilterConfig(threshold=-1)
    with pytest.raises(FilterError):
        vx.FilterConfig(okada_threshold=-0.5)
    with pytest.raises(FilterError):
        vx.FilterConfig(cluster_offset=0)
    with pytest.raises(FilterError, match="none, mean, sigma, okada, entropy, local-cluster"):
        vx.FilterKind.from_name("nosuch")


def test_filter_config_json_digest(vx):
    cfg = vx.FilterConfig(kind=vx.FilterKind.OKADA, kernel_size=5, threshold=101.0,
                          okada_threshold=30.0)
    assert vx.FilterConfig.from_json(cfg.to_json()) == cfg
    a = vx.FilterConfig(kind=vx.FilterKind.MEAN)
    b = vx.FilterConfig(kind=vx.FilterKind.MEAN, threshold=100.0)
    assert a.digest() != b.digest() and len(a.digest()) == 8


def test_resolve_threshold(vx):
    from paper_1807_03119_b200.filters import FilterError

    class H:
        otsu_threshold = 46

    assert vx.FilterConfig().resolve_threshold(H()).threshold == 46.0
    assert vx.FilterConfig(threshold=5.0).resolve_threshold(H()).threshold == 5.0
    with pytest.raises(FilterError, match="histogram"):
        vx.FilterConfig().resolve_threshold(None)


def test_offset_tables_match_reference_definitions():
    from paper_1807_03119_b200.filters import axis_arm_offsets, cluster_offsets, kernel_offsets

    k = kernel_offsets(3)
    assert k.shape == (27, 3) and tuple(k[0]) == (-1, -1, -1) and tuple(k[1]) == (-1, -1, 0)
    assert axis_arm_offsets(3).shape == (9, 3)
    c = cluster_offsets(3, 1)
    assert c.shape == (81, 3)
    assert np.abs(c).max() == 2
    assert kernel_offsets(5).shape == (125, 3)


def test_camera_and_params_validation(vx):
    from paper_1807_03119_b200.render import RenderError

    with pytest.raises(RenderError):
        vx.Camera(position=(0, 0, 10), look_at=(0, 0, 0), up=(0, 0, 1))
    with pytest.raises(RenderError):
        vx.Camera(position=(1, 0, 0), look_at=(0, 0, 0), fov_y_deg=0)
    with pytest.raises(RenderError):
        vx.Camera(position=(1, 0, 0), look_at=(0, 0, 0), fov_y_deg=180)
    with pytest.raises(RenderError):
        vx.RenderParams(width=0)
    with pytest.raises(RenderError):
        vx.RenderParams(step_size=0)
    with pytest.raises(RenderError):
        vx.RenderParams(background=256)
    cam = vx.Camera(position=(10, 4, 7), look_at=(0, 0, 0))
    r, u, f = cam.basis()
    for v in (r, u, f):
        assert np.linalg.norm(v) == pytest.approx(1.0)
    assert vx.Camera.from_json(cam.to_json()) == cam
    p = vx.RenderParams(width=17, light_direction=(0.0, 1.0, 0.0))
    assert vx.RenderParams.from_json(p.to_json()) == p


def test_chunk_rule():
    from paper_1807_03119_b200.render import chunk_for

    assert chunk_for(0.5) == (16, False)
    assert chunk_for(1.0) == (15, False)
    assert chunk_for(2.5) == (6, False)
    assert chunk_for(16.0) == (1, True)
    assert chunk_for(15.0) == (1, False)
    assert chunk_for(14.0) == (1, False)


def test_orbit_camera_matches_oracle(vx, oracle):
    v = vx.Volume(dims=(64, 32, 16), data=np.zeros(64 * 32 * 16, np.uint8))
    cam = vx.orbit_camera(v, azimuth_deg=30, elevation_deg=95)
    pos, look = oracle.orbit((64, 32, 16), 30, 95)
    assert cam.position == pos and cam.look_at == look


def test_volume_validation(vx):
    from paper_1807_03119_b200.volume import VolumeError

    with pytest.raises(VolumeError):
        vx.Volume(dims=(2, 2, 2), data=np.zeros(7, np.uint8))
    with pytest.raises(VolumeError):
        vx.Volume(dims=(0, 2, 2), data=np.zeros(0, np.uint8))
    v = vx.Volume(dims=(3, 2, 1), data=np.arange(6, dtype=np.uint8))
    assert v.sample(2, 1, 0) == 5 and v.sample(3, 0, 0) == 0 and v.sample(-1, 0, 0) == 0
    assert not v.data.flags.writeable


def test_content_hash_matches_reference_definition(vx):
    meta = json.loads((GOLDEN / "phantoms.json").read_text())["spot_64"]
    from oracle.rng_np import generate_phantom_np

    spec = vx.PhantomSpec.from_json(meta["spec"])
    v = vx.Volume(dims=spec.dims, data=generate_phantom_np(spec.to_json()))
    assert v.content_hash() == meta["sha256"]


def test_phantom_specs_match_reference(vx):
    from paper_1807_03119_b200 import phantoms

    meta = json.loads((GOLDEN / "phantoms.json").read_text())
    assert phantoms.spot_phantom_spec(64).to_json() == meta["spot_64"]["spec"]
    assert phantoms.speckle_phantom_spec(128).to_json() == meta["speckle_128"]["spec"]
    assert phantoms.latency_phantom_spec(128).to_json() == meta["latency_128"]["spec"]
    assert phantoms.bench_phantom_spec(128).to_json() == meta["bench_128"]["spec"]


@pytest.mark.skipif(not (GOLDEN / "frames_c2.npz").exists(), reason="C2 fixture not frozen")
def test_insect_spec_is_the_survey_c2_recipe():
    from paper_1807_03119_b200 import phantoms

    g = golden("frames_c2.npz")
    ref = json.loads(str(g["spec_json"]))
    mine = phantoms.insect_phantom_spec(512).to_json()
    assert mine == ref


def test_rng_matches_oracle():
    from oracle import rng_np
    from paper_1807_03119_b200 import rng

    assert rng.substream_seed(20, 0x73706F74) == rng_np.substream_seed(20, 0x73706F74)
    assert np.array_equal(rng.stream(5, 3, 100), rng_np.stream(5, 3, 100))
    a = rng.uniform_indices(123, 500, 1000)
    assert len(set(a.tolist())) == 500 and a.max() < 1000
    assert np.array_equal(a, rng_np.uniform_indices(123, 500, 1000))


def test_native_config_packing(vx):
    from paper_1807_03119_b200.filters import native_config

    counts = np.zeros(256, dtype=np.int64)
    counts[[0, 10, 200]] = [5, 3, 2]

    class H:
        probabilities = counts / counts.sum()
        global_sigma = 12.5

    cfg = vx.FilterConfig(kind=vx.FilterKind.SIGMA, threshold=67.0, sigma_mult=2.0)
    fc = native_config(cfg, H())
    assert fc.kind == 2 and fc.threshold == 67.0 and fc.sigma_band == 25.0
    lut = np.ctypeslib.as_array(fc.entropy_lut)
    p = 0.5
    assert lut[0] == -p * math.log2(p)
    assert lut[1] == 0.0


def test_histogram_validation_messages():
    from paper_1807_03119_b200.histogram import HistogramError, _as_u64_counts

    with pytest.raises(HistogramError, match="expected 256 bins"):
        _as_u64_counts([1, 2, 3])
    with pytest.raises(HistogramError, match="non-negative"):
        _as_u64_counts([-1] + [0] * 255)
    with pytest.raises(HistogramError, match="empty"):
        _as_u64_counts([0] * 256)
    with pytest.raises(HistogramError, match="exact"):
        _as_u64_counts([2 ** 47] + [0] * 255)


def test_frame_header_layout_matches_reference():
    from paper_1807_03119_b200.frames import FRAME_HEADER, pack_frame, unpack_header

    assert FRAME_HEADER.size == 32
    m = pack_frame(3, 640, 480, 1.5, b"ABCDEFGH", b"\x01\x02")
    h = unpack_header(m)
    assert h == {"magic": b"VXSF", "version": 1, "sequence": 3, "width": 640, "height": 480,
                 "render_ms": 1.5, "digest": b"ABCDEFGH"}
    assert m[32:] == b"\x01\x02"


def test_pinned_frame_pool_recycles_only_unreferenced_buffers(monkeypatch):
    """The frame pool hands a page-locked buffer out again only when no array
    or view of it is alive (views of views may reference the flat array or
    the buffer object); double buffering never allocates after warm-up."""
    import ctypes as C

    from paper_1807_03119_b200 import _lib

    keep = []
    allocs = []

    def fake_call(name, *args, **kw):
        assert name == "vx_host_alloc"
        b = (C.c_uint8 * args[0])()
        keep.append(b)
        allocs.append(args[0])
        args[1]._obj.value = C.addressof(b)

    monkeypatch.setattr(_lib, "call", fake_call)
    pool = _lib.PinnedPool()
    for trial in range(4):
        pix, small, p0, p1 = pool.frame(6, 10)
        assert pix.shape == (6, 10) and small.shape == (266,) and p1 - p0 >= 60
        held = [small[:256], pix[1:3], pix.reshape(-1)[2:5], small[256:257].view(np.uint8)][trial]
        del pix, small
        handed = set()
        for _ in range(5):
            q = pool.frame(6, 10)
            handed.add(q[2])
            del q
        assert p0 not in handed
        del held
    n = len(allocs)
    prev = pool.frame(6, 10)
    for _ in range(10):  # render k+1 while frame k is still held
        cur = pool.frame(6, 10)
        assert cur[2] != prev[2]
        prev = cur
    assert len(allocs) == n


def test_pinned_arena_serves_first_frames(monkeypatch):
    """After prewarm() the first frames carve their page-locked buffers from
    the arena (no vx_host_alloc in the frame path); buffers larger than what
    is left fall back to allocation."""
    import ctypes as C

    from paper_1807_03119_b200 import _lib

    keep, allocs = [], []

    def fake_call(name, *args, **kw):
        assert name == "vx_host_alloc"
        b = (C.c_uint8 * args[0])()
        keep.append(b)
        allocs.append(args[0])
        args[1]._obj.value = C.addressof(b)

    monkeypatch.setattr(_lib, "call", fake_call)
    pool = _lib.PinnedPool()
    pool.prewarm()
    pool.prewarm()
    assert allocs == [pool.ARENA_BYTES]
    a = pool.frame(1024, 1024)
    b = pool.frame(1024, 1024)
    # carves are 256-byte aligned relative to the (page-aligned) arena base
    assert len(allocs) == 1 and a[2] != b[2]
    assert (a[2] - pool._arena) % 256 == 0 and (b[2] - pool._arena) % 256 == 0
    # distinct, non-overlapping carves
    lo, hi = sorted([a[2], b[2]])
    assert hi - lo >= 1024 * 1024 + 266 * 8
    big = pool.array((pool.ARENA_BYTES,), np.uint8)  # does not fit the rest: allocated
    assert len(allocs) == 3 and big.size == pool.ARENA_BYTES


def test_pinned_pool_is_bounded(monkeypatch):
    """A client that keeps changing its frame size does not grow page-locked
    memory without bound: at most MAX_FRAME_SIZES sizes keep entries, and
    parked buffers beyond FREE_CAP are freed."""
    import ctypes as C
    import gc

    from paper_1807_03119_b200 import _lib

    keep, allocs, freed = {}, [], []

    def fake_call(name, *args, **kw):
        if name == "vx_host_free":
            freed.append(args[0].value)
            return
        assert name == "vx_host_alloc"
        b = (C.c_uint8 * args[0])()
        keep[C.addressof(b)] = b
        allocs.append(args[0])
        args[1]._obj.value = C.addressof(b)

    monkeypatch.setattr(_lib, "call", fake_call)
    pool = _lib.PinnedPool()
    monkeypatch.setattr(pool, "FREE_CAP", 1 << 20)
    for w in range(40, 80):  # 40 distinct sizes, frames dropped right away
        f = pool.frame(512, w)
        del f
        gc.collect()
    assert len(pool._frames) <= pool.MAX_FRAME_SIZES
    assert pool._free_bytes <= pool.FREE_CAP
    assert freed  # the overflow went back to the driver


def test_pgm_header_grammar(tmp_path):
    """PGM header fields with whitespace / '#'-comment separators, one
    whitespace byte before the payload, and the reference's error messages
    (images.py:20-50)."""
    from paper_1807_03119_b200.images import ImageError, read_pgm, read_pgm_header

    body = bytes(range(12))
    good = [b"P5\n4 3\n255\n", b"P5 4 3 255 ", b"P5\n# c\n4 # x\n3\n#y\n255\n",
            b"P5#c\n4\t3\r255\x0b", b"P5\r\n4\r\n3\r\n255\r"]
    for i, hdr in enumerate(good):
        p = tmp_path / f"g{i}.pgm"
        p.write_bytes(hdr + body)
        assert read_pgm_header(p) == (4, 3, len(hdr))
        assert read_pgm(p).tobytes() == body
    bad = [(b"P6\n4 3\n255\n" + body, "not a binary PGM"), (b"P5\n4 3", "truncated PGM header"),
           (b"P5\n# only a comment", "truncated PGM header"),
           (b"P5\n4 3\n254\n" + body, "maxval must be 255, got 254"),
           (b"P5\n4 3\n255\n" + body[:5], "payload shorter than 4x3")]
    for i, (data, msg) in enumerate(bad):
        p = tmp_path / f"b{i}.pgm"
        p.write_bytes(data)
        with pytest.raises(ImageError, match=msg):
            read_pgm_header(p)
