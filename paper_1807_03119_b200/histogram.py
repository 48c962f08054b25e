"""Grey-level statistics: histogram (K1) and the exact Otsu threshold (K2).

Mirrors histogram.py:26-133 of the reference.  The 256 counts come from the
B200 histogram kernel (computed once when the volume replica is built); the
Otsu argmin runs on the device in exact 320-bit integer arithmetic with the
reference's tie rule (smallest T).  The 256-element derived statistics
(probabilities, population sigma) are evaluated on the host with numpy in the
reference's own operation order so they are bit-identical to it.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .volume import Volume, device_volume

LEVELS = 256


class HistogramError(Exception):
    pass


@dataclass(frozen=True)
class HistogramModel:
    """256-bin histogram with the statistics the filters need (histogram.py:30-56)."""

    counts: np.ndarray
    total: int
    probabilities: np.ndarray
    global_sigma: float
    otsu_threshold: int

    def class_stats(self, t: int | None = None) -> dict:
        t = self.otsu_threshold if t is None else int(t)
        stats = {"threshold": t, "classes": []}
        idx = np.arange(LEVELS, dtype=np.float64)
        for name, sel in (("background", idx <= t), ("data", idx > t)):
            c = self.counts[sel].astype(np.float64)
            n = float(c.sum())
            if n > 0:
                mu = float((c * idx[sel]).sum() / n)
                var = float((c * (idx[sel] - mu) ** 2).sum() / n)
            else:
                mu = var = 0.0
            stats["classes"].append(
                {"name": name, "weight": n / self.total, "count": int(n), "mean": mu, "variance": var}
            )
        return stats


_EXACT_LIMIT = 1 << 47  # N < 2^47 keeps every cross product inside 256 bits


def _as_u64_counts(counts) -> np.ndarray:
    vals = [int(c) for c in counts]
    if len(vals) != LEVELS:
        raise HistogramError(f"expected {LEVELS} bins, got {len(vals)}")
    if any(c < 0 for c in vals):
        raise HistogramError("histogram counts must be non-negative")
    total = sum(vals)
    if total == 0:
        raise HistogramError("histogram is empty (all bins zero)")
    if total >= _EXACT_LIMIT:
        raise HistogramError(
            f"histogram total {total} exceeds the exact device Otsu range (< 2**47)"
        )
    return np.asarray(vals, dtype=np.uint64)


def otsu(counts) -> int:
    """Threshold minimising the weighted intra-class variance (histogram.py:59-101).

    K2 on the B200: exact rational objective per T, compared by 320-bit
    cross-multiplication; ties resolve to the smallest T.
    """
    arr = _as_u64_counts(counts)
    _lib.require_device()
    t = C.c_int32(-1)
    _lib.call("vx_otsu", _lib.ptr(arr), C.byref(t), exc_type=HistogramError)
    if t.value < 0:
        raise HistogramError("device Otsu scan rejected the histogram")
    return int(t.value)


def _sigma_from_counts(counts: np.ndarray) -> float:
    """Population sigma from counts, histogram.py:109-116 operation order."""
    c = counts.astype(np.float64)
    n = c.sum()
    if n == 0:
        raise HistogramError("empty volume")
    idx = np.arange(LEVELS, dtype=np.float64)
    mu = (c * idx).sum() / n
    return float(np.sqrt((c * (idx - mu) ** 2).sum() / n))


def volume_counts(volume: Volume) -> np.ndarray:
    """K1 counts of the volume (int64[256]) from its device replica."""
    return device_volume(volume).counts()


def global_stddev(volume: Volume) -> float:
    """Population standard deviation of all voxel intensities (histogram.py:104-106)."""
    return _sigma_from_counts(volume_counts(volume))


def model_from_counts(counts: np.ndarray) -> HistogramModel:
    counts = np.asarray(counts, dtype=np.int64).copy()
    total = int(counts.sum())
    if total == 0:
        raise HistogramError("empty volume")
    counts.flags.writeable = False
    probabilities = counts / total
    probabilities.flags.writeable = False
    return HistogramModel(
        counts=counts,
        total=total,
        probabilities=probabilities,
        global_sigma=_sigma_from_counts(counts),
        otsu_threshold=otsu(counts),
    )


def build_histogram(volume: Volume) -> HistogramModel:
    """Histogram + Otsu of a volume (histogram.py:119-133) via K1/K2."""
    return model_from_counts(volume_counts(volume))


def histogram_of_bytes(data: np.ndarray) -> np.ndarray:
    """K1 over an arbitrary host uint8 buffer (uploaded)."""
    _lib.require_device()
    arr = np.ascontiguousarray(data, dtype=np.uint8).reshape(-1)
    out = np.zeros(LEVELS, dtype=np.uint64)
    _lib.call("vx_histogram_host", _lib.ptr(arr), arr.size, _lib.ptr(out))
    return out.astype(np.int64)
