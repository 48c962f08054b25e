"""Counter-mode splitmix64 draws (host side of the phantom input generator).

Same stream definition as the reference (rng.py:1-73): draw ``j`` of seed
``s`` is ``mix64(s + (j + 1) * 0x9E3779B97F4A7C15)`` modulo 2**64.  Only the
pieces the host needs are here: stream draws for blob placement and the
distinct spot indices; the per-voxel Gaussian noise runs on the device
(csrc/vx_volume.cu noise_kernel).
"""

from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK = 0xFFFFFFFFFFFFFFFF


def mix64(x):
    """splitmix64 finaliser (rng.py:24-30)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64)
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def stream(seed: int, start: int, count: int) -> np.ndarray:
    """Draws start .. start+count-1 (rng.py:33-38)."""
    j = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(np.uint64(seed & _MASK) + (j + np.uint64(1)) * GOLDEN)


def substream_seed(seed: int, tag: int) -> int:
    """Independent stream seed for (seed, tag) (rng.py:41-43)."""
    return int(mix64(np.uint64((seed ^ tag) & _MASK)))


def uniform_indices(seed: int, k: int, n: int) -> np.ndarray:
    """First k distinct values of ``draw mod n`` in draw order (rng.py:54-73)."""
    if k > n:
        raise ValueError(f"cannot draw {k} distinct indices from {n}")
    picked: list[int] = []
    seen: set[int] = set()
    start = 0
    while len(picked) < k:
        batch = max(256, 2 * (k - len(picked)))
        for v in (stream(seed, start, batch) % np.uint64(n)).tolist():
            if v not in seen:
                seen.add(v)
                picked.append(v)
                if len(picked) == k:
                    break
        start += batch
    return np.asarray(picked, dtype=np.int64)
