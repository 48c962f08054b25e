"""K1 histogram, K2 exact Otsu, K6 image entropy on the B200 vs the oracle and
the reference's golden vectors (mirrors tests/test_histogram.py and
tests/test_metrics.py of the reference)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def make_volume(vx, values):
    arr = np.asarray(values, dtype=np.uint8)
    return vx.Volume(dims=(arr.size, 1, 1), data=arr)


@pytest.mark.parametrize("n", [1, 7, 15, 16, 17, 255, 4096 + 3, 1 << 20, (1 << 24) + 11])
def test_k1_histogram_sizes(vx, oracle, n):
    from paper_1807_03119_b200.histogram import histogram_of_bytes

    rs = np.random.default_rng(n)
    data = rs.integers(0, 256, n, dtype=np.uint8)
    assert np.array_equal(histogram_of_bytes(data), oracle.hist256(data))


def _fused(t, n, stream=None):
    """vx_histogram_otsu_device (K1+K2 in one launch) over device bytes."""
    import ctypes as C

    import torch

    from paper_1807_03119_b200 import _lib

    s = stream or torch.cuda.current_stream()
    counts = torch.full((256,), -1, dtype=torch.int64, device="cuda")
    T = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    _lib.call("vx_histogram_otsu_device", C.c_void_p(t.data_ptr() if n else 0), n,
              C.c_void_p(counts.data_ptr()), C.c_void_p(T.data_ptr()), C.c_void_p(s.cuda_stream))
    return counts, T


@pytest.mark.parametrize("n", [0, 1, 7, 16, 17, 4096 + 3, 1 << 20, (1 << 24) + 11, (1 << 27) + 5])
def test_fused_hist_otsu_sizes(vx, oracle, n):
    """One-launch K1+K2: counts bit-exact, T equal to the exact oracle Otsu;
    back-to-back calls on one stream (the workspace resets itself) and on a
    second stream agree."""
    import torch

    rs = np.random.default_rng(n + 3)
    host = rs.integers(0, 256, n, dtype=np.uint8)
    host[: n // 2] = rs.integers(0, 30, n // 2, dtype=np.uint8)  # bimodal-ish
    t = torch.from_numpy(host).cuda()
    want = oracle.hist256(host)
    want_T = oracle.otsu(want) if n else -1
    side = torch.cuda.Stream()
    for rep in range(3):
        for s in (None, side):
            off = 3 if (rep == 2 and n > 3) else 0  # unaligned start
            sub = t[off:]
            counts, T = _fused(sub, n - off, s)
            torch.cuda.synchronize()
            w = want if off == 0 else oracle.hist256(host[off:])
            assert np.array_equal(counts.cpu().numpy(), w)
            wt = want_T if off == 0 else (oracle.otsu(w) if n - off else -1)
            assert int(T.item()) == wt


def test_fused_hist_otsu_concurrent_streams(vx, oracle):
    """Four streams launching K1+K2 at once, several rounds without a host
    sync in between: each launch has its own Otsu block waiting on its own
    counting blocks (per-stream workspaces), none waits on another's."""
    import torch

    rs = np.random.default_rng(11)
    hosts = [rs.integers(0, 256, (1 << 24) + 7 * i, dtype=np.uint8) for i in range(4)]
    for h in hosts:
        h[: h.size // 3] = rs.integers(0, 40, h.size // 3, dtype=np.uint8)
    import ctypes as C

    from paper_1807_03119_b200 import _lib

    devs = [torch.from_numpy(h).cuda() for h in hosts]
    streams = [torch.cuda.Stream() for _ in hosts]
    outs = [[(torch.full((256,), -1, dtype=torch.int64, device="cuda"),
              torch.full((1,), -7, dtype=torch.int32, device="cuda")) for _ in hosts]
            for _ in range(3)]
    torch.cuda.synchronize()
    for rnd in outs:  # launches only: no torch work between them
        for d, s, (counts, T) in zip(devs, streams, rnd):
            _lib.call("vx_histogram_otsu_device", C.c_void_p(d.data_ptr()), d.numel(),
                      C.c_void_p(counts.data_ptr()), C.c_void_p(T.data_ptr()),
                      C.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    for rnd in outs:
        for h, (counts, T) in zip(hosts, rnd):
            want = oracle.hist256(h)
            assert np.array_equal(counts.cpu().numpy(), want)
            assert int(T.item()) == oracle.otsu(want)


def test_fused_hist_otsu_goldens(vx, oracle):
    """The reference's golden Otsu histograms, expanded to bytes where small."""
    import torch

    g = golden("otsu.npz")
    done = 0
    for counts, thr in zip(g["counts"], g["threshold"]):
        if int(np.sum(counts)) > (1 << 22):
            continue
        host = np.repeat(np.arange(256, dtype=np.uint8), np.asarray(counts, dtype=np.int64))
        np.random.default_rng(done).shuffle(host)
        c, T = _fused(torch.from_numpy(host).cuda(), host.size)
        torch.cuda.synchronize()
        assert np.array_equal(c.cpu().numpy(), counts)
        assert int(T.item()) == thr
        done += 1
        if done == 200:
            break
    assert done >= 50


def test_k1_unaligned_and_skewed(vx, oracle):
    from paper_1807_03119_b200.histogram import histogram_of_bytes

    rs = np.random.default_rng(1)
    buf = rs.integers(0, 256, (1 << 22) + 64, dtype=np.uint8)
    buf[: 3 << 20] = 0  # CT-like background spike
    for off in (0, 1, 3, 15):
        view = buf[off:off + (1 << 22) - 5]
        assert np.array_equal(histogram_of_bytes(view), oracle.hist256(view))
    assert np.array_equal(histogram_of_bytes(np.full(1 << 21, 255, np.uint8)),
                          oracle.hist256(np.full(1 << 21, 255, np.uint8)))


def test_build_histogram_models(vx):
    h = vx.build_histogram(make_volume(vx, [5] * 8))
    assert h.counts[5] == 8 and h.total == 8 and h.probabilities[5] == 1.0
    assert h.global_sigma == 0.0
    h = vx.build_histogram(make_volume(vx, [0] * 4 + [255] * 4))
    assert h.probabilities[0] == 0.5 and h.global_sigma == 127.5
    h = vx.build_histogram(make_volume(vx, list(range(200))))
    assert h.total == 200 and abs(h.probabilities.sum() - 1.0) < 1e-9
    assert vx.global_stddev(make_volume(vx, [0, 0, 0, 4])) == pytest.approx(math.sqrt(3))


def test_k2_otsu_reference_goldens(vx):
    g = golden("otsu.npz")
    for counts, t in zip(g["counts"], g["threshold"]):
        assert vx.otsu(counts) == t


def test_k2_otsu_known_answers_and_errors(vx):
    from paper_1807_03119_b200.histogram import HistogramError

    c = [0] * 256
    c[10] = c[200] = 500
    assert vx.otsu(c) == 10
    c = [0] * 256
    c[137] = 42
    assert vx.otsu(c) == 0
    c = [0] * 256
    c[100] = c[101] = 10
    assert vx.otsu(c) == 100
    with pytest.raises(HistogramError):
        vx.otsu([0] * 256)
    with pytest.raises(HistogramError):
        vx.otsu([1] * 255)


def test_k2_otsu_scale_invariance_and_big_counts(vx, oracle):
    rs = np.random.default_rng(9)
    for _ in range(20):
        counts = [int(v) for v in rs.integers(0, 50, 256)]
        k = int(rs.integers(1, 10000))
        assert vx.otsu(counts) == vx.otsu([k * v for v in counts]) == oracle.otsu(counts)
    # 4096^3-sized histograms: 2^36 voxels need the 320-bit compare
    for _ in range(10):
        counts = rs.integers(0, 2 ** 28, 256)
        counts[0] = 2 ** 35
        assert vx.otsu(counts) == oracle.otsu(counts)


def test_image_entropy(vx, oracle):
    g = golden("shading.npz")
    for i in range(4):
        assert vx.image_entropy(g[f"img{i}"]) == pytest.approx(float(g[f"img{i}_H"]), abs=1e-12)
    assert vx.image_entropy(np.full((8, 8), 77, np.uint8)) == 0.0
    img = np.zeros((4, 4), np.uint8)
    img[:2] = 255
    assert vx.image_entropy(img) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        vx.image_entropy(np.zeros((0, 4), np.uint8))
    rs = np.random.default_rng(5)
    for _ in range(10):
        im = rs.integers(0, 256, (64, 48), dtype=np.uint8)
        assert vx.image_entropy(im) == pytest.approx(oracle.image_entropy(im), abs=1e-12)
