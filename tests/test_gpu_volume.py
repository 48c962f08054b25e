"""K3 volume ingestion (load_raw 8/16-bit, slice stacks), the device replica,
the exact-skip distance map and the K7 phantom generator (mirrors
tests/test_volume.py of the reference)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu


def test_load_raw_8bit_roundtrip(vx, tmp_path):
    rs = np.random.default_rng(1)
    v = vx.Volume(dims=(7, 5, 3), data=rs.integers(0, 256, 105, dtype=np.uint8))
    vx.save_raw(v, tmp_path / "a.raw")
    w = vx.load_raw(tmp_path / "a.raw")
    assert w.dims == (7, 5, 3) and np.array_equal(w.data, v.data)
    from paper_1807_03119_b200.volume import device_volume

    assert np.array_equal(device_volume(w).read(), v.data)


def test_load_raw_16bit_rescale_exhaustive(vx, tmp_path):
    g = golden("shading.npz")
    wide = np.arange(65536, dtype="<u2")
    (tmp_path / "w.raw").write_bytes(wide.tobytes())
    meta = vx.VolumeMeta(dims=(256, 256, 1), bit_depth=16)
    v = vx.load_raw(tmp_path / "w.raw", meta)
    assert np.array_equal(v.data.reshape(-1), g["u16_rescale"])
    # histogram of the rescaled volume is the device one
    assert np.array_equal(vx.build_histogram(v).counts, np.bincount(g["u16_rescale"], minlength=256))


def test_load_raw_errors(vx, tmp_path):
    from paper_1807_03119_b200.volume import VolumeError

    (tmp_path / "b.raw").write_bytes(b"\0" * 10)
    with pytest.raises(VolumeError, match="expected 8 bytes.*file has 10"):
        vx.load_raw(tmp_path / "b.raw", vx.VolumeMeta(dims=(2, 2, 2)))
    with pytest.raises(FileNotFoundError):
        vx.load_raw(tmp_path / "nope.raw")
    with pytest.raises(VolumeError):
        vx.load_raw(tmp_path / "b.raw")


def test_slice_stack(vx, tmp_path):
    from paper_1807_03119_b200.images import write_pgm

    rs = np.random.default_rng(2)
    slices = rs.integers(0, 256, (4, 6, 5), dtype=np.uint8)
    for i, s in enumerate(slices):
        write_pgm(s, tmp_path / f"s{i:02d}.pgm")
    v = vx.load_slice_stack(tmp_path)
    assert v.dims == (5, 6, 4) and np.array_equal(v.data, slices)


@pytest.mark.parametrize("bits", [8, 16])
def test_streamed_ingest_multi_chunk(vx, tmp_path, monkeypatch, bits):
    """§8f2: the direct-to-device loader over many 1 MiB chunks (slot
    wrap-around, u16 chunks rescaled on the device) equals numpy's load."""
    monkeypatch.setenv("VOXB200_IO_CHUNK_MB", "1")
    rs = np.random.default_rng(bits)
    dims = (96, 80, 70)
    n = dims[0] * dims[1] * dims[2]
    if bits == 8:
        raw = rs.integers(0, 256, n, dtype=np.uint8)
        want = raw
    else:
        raw = rs.integers(0, 65536, n, dtype=np.uint32).astype("<u2")
        want = ((raw.astype(np.int64) + 128) // 257).astype(np.uint8)
    raw.tofile(tmp_path / "v.raw")
    v = vx.load_raw(tmp_path / "v.raw", vx.VolumeMeta(dims=dims, bit_depth=bits))
    assert np.array_equal(v.data.reshape(-1), want)
    from paper_1807_03119_b200.volume import device_volume

    dv = device_volume(v)
    assert np.array_equal(dv.read().reshape(-1), want)
    assert np.array_equal(dv.counts(), np.bincount(want, minlength=256))


def test_streamed_slice_stack_straddles_chunks(vx, tmp_path, monkeypatch):
    from paper_1807_03119_b200.images import write_pgm
    from paper_1807_03119_b200.volume import VolumeError, device_volume

    monkeypatch.setenv("VOXB200_IO_CHUNK_MB", "1")
    rs = np.random.default_rng(3)
    slices = rs.integers(0, 256, (23, 301, 197), dtype=np.uint8)  # 59 KB slices
    for i, sl in enumerate(slices):
        write_pgm(sl, tmp_path / f"z{i:03d}.pgm")
    # a comment in one header moves its payload offset
    (tmp_path / "z005.pgm").write_bytes(b"P5\n# scanner 7\n197 301\n255\n" + slices[5].tobytes())
    v = vx.load_slice_stack(tmp_path)
    assert v.dims == (197, 301, 23) and np.array_equal(v.data, slices)
    assert np.array_equal(device_volume(v).read(), slices)
    (tmp_path / "z010.pgm").write_bytes(b"P5\n197 301\n255\n" + slices[10].tobytes()[:-1])
    with pytest.raises(VolumeError, match="payload shorter than 197x301"):
        vx.load_slice_stack(tmp_path)
    (tmp_path / "z010.pgm").write_bytes(b"P5\n196 301\n255\n" + slices[10].tobytes())
    with pytest.raises(VolumeError, match="slice is 196x301, previous slices are 197x301"):
        vx.load_slice_stack(tmp_path)


@pytest.mark.parametrize("name", ["spot_64", "latency_64", "latency_128", "bench_128"])
def test_device_phantom_matches_reference_bytes(vx, name):
    meta = json.loads((GOLDEN / "phantoms.json").read_text())[name]
    spec = vx.PhantomSpec.from_json(meta["spec"])
    v = vx.generate_phantom(spec)
    assert v.content_hash() == meta["sha256"]


def test_device_phantom_vs_oracle_generator_256(vx, oracle):
    from paper_1807_03119_b200 import phantoms

    spec = phantoms.insect_phantom_spec(256)
    v = vx.generate_phantom(spec)
    ref = oracle.phantom(spec.to_json(), threads=oracle.max_threads())
    assert int((v.data != ref).sum()) == 0


def _brute_distance(bmax_occ: np.ndarray, cap: int) -> np.ndarray:
    occ = np.argwhere(bmax_occ)
    mz, my, mx = bmax_occ.shape
    out = np.full(bmax_occ.shape, cap, dtype=np.int64)
    if len(occ) == 0:
        return out
    zz, yy, xx = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    for oz, oy, ox in occ:
        d = np.maximum(np.maximum(abs(zz - oz), abs(yy - oy)), abs(xx - ox))
        out = np.minimum(out, d)
    return out


def _separable_distance(occ: np.ndarray, cap: int) -> np.ndarray:
    """Chebyshev distance (capped) by the separable min-max passes, in numpy."""
    big = np.int64(cap)
    d = np.where(occ, 0, big).astype(np.int64)
    for axis in (2, 1, 0):  # x, y, z
        n = d.shape[axis]
        out = np.full(d.shape, big, dtype=np.int64)
        for k in range(-cap + 1, cap):
            if abs(k) >= n:
                continue
            src = [slice(None)] * 3
            dst = [slice(None)] * 3
            if k >= 0:
                src[axis], dst[axis] = slice(k, n), slice(0, n - k)
            else:
                src[axis], dst[axis] = slice(0, n + k), slice(-k, n)
            out[tuple(dst)] = np.minimum(out[tuple(dst)], np.maximum(d[tuple(src)], abs(k)))
        d = out
    return d


def test_distance_map_long_lines(vx):
    """Fine (4^3, cap 32) and coarse (8^3, cap 24) maps of a volume whose cell
    lines are longer than twice the cap, against a numpy restatement; sparse
    points, a slab and a line of occupied cells."""
    from paper_1807_03119_b200.volume import device_volume

    rs = np.random.default_rng(7)
    nz, ny, nx = 300, 272, 264
    data = rs.integers(0, 90, (nz, ny, nx), dtype=np.uint8)
    for _ in range(25):
        data[rs.integers(0, nz), rs.integers(0, ny), rs.integers(0, nx)] = 210
    data[150:160, 20:30, 100:240] = 180
    data[5, 250, :] = 255
    dv = device_volume(vx.Volume(dims=(nx, ny, nz), data=data))
    caps = {lv: dv.skip_cap(lv) for lv in (0, 1)}
    for c, cap, level in ((4, caps[1], 1), (8, caps[0], 0)):
        ncz, ncy, ncx = (nz + c - 1) // c, (ny + c - 1) // c, (nx + c - 1) // c
        pad = np.zeros((ncz * c, ncy * c, ncx * c), dtype=np.uint8)
        pad[:nz, :ny, :nx] = data
        cmax = pad.reshape(ncz, c, ncy, c, ncx, c).max(axis=(1, 3, 5))
        for thr in (100, 200):
            occ = np.zeros((ncz + 2, ncy + 2, ncx + 2), dtype=bool)
            occ[1:-1, 1:-1, 1:-1] = cmax >= thr
            got = dv.distance_map(thr, level=level).astype(np.int64)
            assert np.array_equal(got, _separable_distance(occ, cap)), (c, thr)


def test_distance_map_is_exact_chebyshev(vx):
    from paper_1807_03119_b200.volume import device_volume

    rs = np.random.default_rng(4)
    data = rs.integers(0, 50, (70, 41, 33), dtype=np.uint8)
    for _ in range(12):
        z, y, x = rs.integers(0, 70), rs.integers(0, 41), rs.integers(0, 33)
        data[z, y, x] = 200
    v = vx.Volume(dims=(33, 41, 70), data=data)
    dv = device_volume(v)
    dm = dv.distance_map(100).astype(np.int64)
    nbz, nby, nbx = (70 + 7) // 8, (41 + 7) // 8, (33 + 7) // 8
    pad = np.zeros((nbz * 8, nby * 8, nbx * 8), dtype=np.uint8)
    pad[:70, :41, :33] = data
    bmax = pad.reshape(nbz, 8, nby, 8, nbx, 8).max(axis=(1, 3, 5))
    occ = np.zeros((nbz + 2, nby + 2, nbx + 2), dtype=bool)
    occ[1:-1, 1:-1, 1:-1] = bmax >= 100
    want = _brute_distance(occ, dv.skip_cap(0))
    assert np.array_equal(dm, want)
    # fine level: 4^3 cells, cap 32
    fm = dv.distance_map(100, level=1).astype(np.int64)
    c = 4
    ncz, ncy, ncx = (70 + c - 1) // c, (41 + c - 1) // c, (33 + c - 1) // c
    pad2 = np.zeros((ncz * c, ncy * c, ncx * c), dtype=np.uint8)
    pad2[:70, :41, :33] = data
    cmax = pad2.reshape(ncz, c, ncy, c, ncx, c).max(axis=(1, 3, 5))
    occ2 = np.zeros((ncz + 2, ncy + 2, ncx + 2), dtype=bool)
    occ2[1:-1, 1:-1, 1:-1] = cmax >= 100
    assert np.array_equal(fm, _brute_distance(occ2, dv.skip_cap(1)))


def _brute_orthant(occ: np.ndarray, cap: int, oct: int) -> np.ndarray:
    """min over occupied o with s_a (o_a - c_a) >= 0 (s_a = -1 if bit a of
    oct, axes x, y, z) of max_a s_a (o_a - c_a), capped."""
    sx, sy, sz = (-1 if (oct >> a) & 1 else 1 for a in range(3))
    mz, my, mx = occ.shape
    zz, yy, xx = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    out = np.full(occ.shape, cap, dtype=np.int64)
    for oz, oy, ox in np.argwhere(occ):
        dx, dy, dz = sx * (ox - xx), sy * (oy - yy), sz * (oz - zz)
        ok = (dx >= 0) & (dy >= 0) & (dz >= 0)
        d = np.where(ok, np.maximum(np.maximum(dx, dy), dz), cap)
        out = np.minimum(out, d)
    return np.minimum(out, cap)


def test_orthant_maps_exact(vx):
    """The eight orthant skip maps equal a brute-force one-sided Chebyshev
    distance over the 4^3 cells (including lines longer than the cap)."""
    from paper_1807_03119_b200.volume import device_volume

    rs = np.random.default_rng(7)
    data = rs.integers(0, 50, (150, 37, 29), dtype=np.uint8)
    for _ in range(9):
        z, y, x = rs.integers(0, 150), rs.integers(0, 37), rs.integers(0, 29)
        data[z, y, x] = 220
    v = vx.Volume(dims=(29, 37, 150), data=data)
    dv = device_volume(v)
    c = 4
    ncz, ncy, ncx = (150 + c - 1) // c, (37 + c - 1) // c, (29 + c - 1) // c
    pad = np.zeros((ncz * c, ncy * c, ncx * c), dtype=np.uint8)
    pad[:150, :37, :29] = data
    cmax = pad.reshape(ncz, c, ncy, c, ncx, c).max(axis=(1, 3, 5))
    occ = np.zeros((ncz + 2, ncy + 2, ncx + 2), dtype=bool)
    occ[1:-1, 1:-1, 1:-1] = cmax >= 100
    iso = dv.distance_map(100, level=1).astype(np.int64)
    for o in range(8):
        got = dv.distance_map(100, level=8 + o).astype(np.int64)
        want = _brute_orthant(occ, dv.skip_cap(1), o)
        assert np.array_equal(got, want), o
        assert np.all(got >= iso)  # one-sided: never shorter than the two-sided map


def test_long_volume_uses_a_larger_cap_exactly(vx):
    """A 2100-voxel-long volume gets the 128-cell cap (vx_fine_cap_for): its
    two-sided and orthant maps are still the exact capped distances."""
    from paper_1807_03119_b200.volume import device_volume

    rs = np.random.default_rng(11)
    nz, ny, nx = 2100, 12, 10
    data = rs.integers(0, 40, (nz, ny, nx), dtype=np.uint8)
    for z in (3, 700, 1500, 2099):
        data[z, rs.integers(0, ny), rs.integers(0, nx)] = 240
    dv = device_volume(vx.Volume(dims=(nx, ny, nz), data=data))
    cap = dv.skip_cap(1)
    assert cap == 128
    c = 4
    ncz, ncy, ncx = (nz + c - 1) // c, (ny + c - 1) // c, (nx + c - 1) // c
    pad = np.zeros((ncz * c, ncy * c, ncx * c), dtype=np.uint8)
    pad[:nz, :ny, :nx] = data
    cmax = pad.reshape(ncz, c, ncy, c, ncx, c).max(axis=(1, 3, 5))
    occ = np.zeros((ncz + 2, ncy + 2, ncx + 2), dtype=bool)
    occ[1:-1, 1:-1, 1:-1] = cmax >= 100
    assert np.array_equal(dv.distance_map(100, level=1).astype(np.int64),
                          _brute_distance(occ, cap).clip(max=cap))
    for o in (0, 4, 7):
        assert np.array_equal(dv.distance_map(100, level=8 + o).astype(np.int64),
                              _brute_orthant(occ, cap, o)), o
