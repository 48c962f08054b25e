"""K5 filters on the B200 vs the reference's golden values (mirrors
tests/test_filters.py of the reference): exact equality, not tolerance."""

from __future__ import annotations

import itertools

import numpy as np
import pytest

from conftest import golden, vol_from

pytestmark = pytest.mark.gpu


def constant(vx, v, n=9):
    return vol_from(vx, np.full((n, n, n), v, dtype=np.uint8))


def test_reference_golden_filter_values(vx):
    from paper_1807_03119_b200.filters import apply_filter, apply_filter_batch

    g = golden("filters.npz")
    kinds = {k.value: k for k in vx.FilterKind}
    for vol, pts, kind, m, d, sc, bt in zip(g["volumes"], g["coords"], g["kinds"], g["kernel"],
                                            g["offset"], g["scalar"], g["batch"]):
        v = vx.Volume(dims=(9, 9, 9), data=vol)
        h = vx.build_histogram(v)
        cfg = vx.FilterConfig(kind=kinds[str(kind)], kernel_size=int(m), cluster_offset=int(d))
        got = apply_filter_batch(v, pts[:, 0], pts[:, 1], pts[:, 2], cfg, h)
        assert np.array_equal(got, bt), (kind, m, d)
        got_s = np.array([apply_filter(v, *map(int, p), cfg, h) for p in pts])
        assert np.array_equal(got_s, sc), (kind, m, d)


def test_local_cluster_goldens(vx, spot_volume):
    from paper_1807_03119_b200.filters import FilterError, local_cluster_filter

    cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER)
    assert local_cluster_filter(constant(vx, 123), 4, 4, 4, cfg) == 123.0
    assert local_cluster_filter(spot_volume, 4, 4, 4, cfg) == pytest.approx(255 / 27)
    data = np.zeros((9, 9, 9), dtype=np.uint8)
    data[:, :, :5] = 200
    assert local_cluster_filter(vol_from(vx, data), 4, 4, 4, cfg) == pytest.approx(3200 / 27)
    with pytest.raises(FilterError):
        local_cluster_filter(spot_volume, 4, 4, 4, vx.FilterConfig(kind=vx.FilterKind.MEAN))


def test_axis_mean_sigma_okada_entropy_goldens(vx):
    from paper_1807_03119_b200.filters import (axis_cluster_average, entropy_filter, mean_filter,
                                               okada_filter, sigma_filter)

    assert axis_cluster_average(constant(vx, 90), 4, 4, 4) == 90.0
    data = np.full((9, 9, 9), 30, dtype=np.uint8)
    data[4, 4, 4] = 0
    assert axis_cluster_average(vol_from(vx, data), 4, 4, 4) == pytest.approx(20.0)
    assert mean_filter(constant(vx, 44), 4, 4, 4) == 44.0
    assert mean_filter(constant(vx, 27), 0, 0, 0) == pytest.approx(8.0)
    data = np.full((9, 9, 9), 10, dtype=np.uint8)
    data[4, 4, 4] = 200
    assert sigma_filter(vol_from(vx, data), 4, 4, 4, 3, 2.0, 0.0) == 200.0
    assert sigma_filter(vol_from(vx, data), 4, 4, 4, 3, 2.0, 5.0) == 200.0
    data[4, 4, 4] = 37
    assert sigma_filter(vol_from(vx, data), 4, 4, 4, 3, 2.0, 200.0) == pytest.approx((26 * 10 + 37) / 27)
    data = np.full((9, 9, 9), 250, dtype=np.uint8)
    data[4, 4, 4] = 100
    assert okada_filter(vol_from(vx, data), 4, 4, 4, 5.0) == 0.0
    data[4, 4, 3] = 98
    data[4, 4, 5] = 99
    assert okada_filter(vol_from(vx, data), 4, 4, 4, 5.0) == pytest.approx(98.5)
    data = np.zeros((6, 6, 6), dtype=np.uint8)
    data[:3] = 7
    data[3:] = 9
    v = vol_from(vx, data)
    h = vx.build_histogram(v)
    assert entropy_filter(v, 3, 3, 3, 3, 13.4, h.probabilities) != 0.0
    assert entropy_filter(v, 3, 3, 3, 3, 13.6, h.probabilities) == 0.0
    c = constant(vx, 77)
    assert entropy_filter(c, 4, 4, 4, 3, -1.0, vx.build_histogram(c).probabilities) == 77.0


def test_missing_histogram_is_config_error(vx, constant_volume):
    from paper_1807_03119_b200.filters import FilterError, apply_filter

    for kind in (vx.FilterKind.SIGMA, vx.FilterKind.ENTROPY):
        with pytest.raises(FilterError, match="histogram"):
            apply_filter(constant_volume, 4, 4, 4, vx.FilterConfig(kind=kind))


def test_filters_vs_oracle_random(vx, oracle):
    from paper_1807_03119_b200.filters import apply_filter_batch

    rs = np.random.default_rng(11)
    for trial in range(10):
        data = rs.integers(0, 256, (11, 13, 9), dtype=np.uint8)
        v = vol_from(vx, data)
        h = vx.build_histogram(v)
        pts = rs.integers(-3, 15, (64, 3))
        for kind in vx.FilterKind:
            for m, d in ((3, 1), (5, 2), (7, 1)):
                cfg = vx.FilterConfig(kind=kind, kernel_size=m, cluster_offset=d)
                got = apply_filter_batch(v, pts[:, 0], pts[:, 1], pts[:, 2], cfg, h)
                want = oracle.filter_batch(data, pts[:, 0], pts[:, 1], pts[:, 2], kind=kind.value,
                                           kernel_size=m, cluster_offset=d,
                                           sigma_band=2.0 * h.global_sigma,
                                           probabilities=h.probabilities, pairwise=False)
                assert np.array_equal(got, want), (kind, m, d)


def test_axis_symmetry_invariance(vx):
    from paper_1807_03119_b200.filters import apply_filter

    n = 7
    rs = np.random.default_rng(8)
    data = rs.integers(0, 256, (n, n, n), dtype=np.uint8)
    v = vol_from(vx, data)
    h = vx.build_histogram(v)
    coord = (2, 3, 4)
    expected = {k: apply_filter(v, *coord, vx.FilterConfig(kind=k), h) for k in vx.FilterKind}
    for perm in itertools.permutations(range(3)):
        for flips in itertools.product((False, True), repeat=3):
            new = np.zeros_like(data)
            zz, yy, xx = np.meshgrid(range(n), range(n), range(n), indexing="ij")
            p = np.stack([xx, yy, zz])
            q = np.stack([p[perm[a]] for a in range(3)])
            q = np.stack([(n - 1 - q[a]) if flips[a] else q[a] for a in range(3)])
            new[q[2], q[1], q[0]] = data
            tv = vol_from(vx, new)
            th = vx.build_histogram(tv)
            c = [coord[perm[a]] for a in range(3)]
            tc = tuple((n - 1 - c[a]) if flips[a] else c[a] for a in range(3))
            for kind in vx.FilterKind:
                got = apply_filter(tv, *tc, vx.FilterConfig(kind=kind), th)
                assert got == pytest.approx(expected[kind], abs=1e-9), (kind, perm, flips)
