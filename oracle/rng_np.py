"""splitmix64 counter-mode draws (restates rng.py:24-73) — test infrastructure only.

Also holds ``generate_phantom_np``: a numpy restatement of generate_phantom
(volume.py:317-368) that is bit-identical to the reference on the same numpy
(pinned by the phantom sha256 fixtures in tests/golden/).
"""

from __future__ import annotations

import math

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(x):
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64)
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def stream(seed, start, count):
    j = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (j + np.uint64(1)) * _G)


def substream_seed(seed, tag):
    return int(mix64(np.uint64((seed ^ tag) & 0xFFFFFFFFFFFFFFFF)))


def gaussian(seed, count):
    bits = stream(seed, 0, 2 * count)
    u1 = ((bits[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (bits[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def uniform_indices(seed, k, n):
    seen, out, start = set(), [], 0
    while len(out) < k:
        batch = max(256, 2 * (k - len(out)))
        for v in (stream(seed, start, batch) % np.uint64(n)).tolist():
            if v not in seen:
                seen.add(v)
                out.append(v)
                if len(out) == k:
                    break
        start += batch
    return np.asarray(out, dtype=np.int64)


def generate_phantom_np(spec: dict) -> np.ndarray:
    """(nz, ny, nx) uint8 volume from spec.to_json() (volume.py:317-368)."""
    nx, ny, nz = (int(v) for v in spec["dims"])
    n = nx * ny * nz
    base = np.zeros((nz, ny, nx), dtype=np.float64)
    for s in spec.get("shapes", []):
        cx, cy, cz = s["center"]
        if s["kind"] == "box":
            rx, ry, rz = (e / 2.0 for e in s["extent"])
        else:
            r = s["radius"] + (s.get("thickness", 0.0) / 2.0 if s["kind"] == "shell" else 0.0)
            rx = ry = rz = r
        x0, x1 = max(0, math.ceil(cx - rx)), min(nx - 1, math.floor(cx + rx))
        y0, y1 = max(0, math.ceil(cy - ry)), min(ny - 1, math.floor(cy + ry))
        z0, z1 = max(0, math.ceil(cz - rz)), min(nz - 1, math.floor(cz + rz))
        if x0 > x1 or y0 > y1 or z0 > z1:
            continue
        xs = np.arange(x0, x1 + 1, dtype=np.float64)[None, None, :]
        ys = np.arange(y0, y1 + 1, dtype=np.float64)[None, :, None]
        zs = np.arange(z0, z1 + 1, dtype=np.float64)[:, None, None]
        if s["kind"] == "sphere":
            inside = (xs - cx) ** 2 + (ys - cy) ** 2 + (zs - cz) ** 2 <= s["radius"] ** 2
        elif s["kind"] == "shell":
            d2 = (xs - cx) ** 2 + (ys - cy) ** 2 + (zs - cz) ** 2
            inside = np.abs(np.sqrt(d2) - s["radius"]) <= s["thickness"] / 2.0
        else:
            ex, ey, ez = s["extent"]
            inside = ((np.abs(xs - cx) <= ex / 2.0) & (np.abs(ys - cy) <= ey / 2.0)
                      & (np.abs(zs - cz) <= ez / 2.0))
        base[z0:z1 + 1, y0:y1 + 1, x0:x1 + 1][inside] = float(s["intensity"])
    sigma = float(spec.get("noise", {}).get("sigma", 0.0))
    seed = int(spec.get("rng_seed", 0))
    if sigma > 0:
        z = gaussian(substream_seed(seed, 0x6E6F697365), n).reshape(nz, ny, nx)
        base = np.floor(base + sigma * z + 0.5)
    out = np.clip(base, 0.0, 255.0).astype(np.uint8)
    spot = spec.get("spot_noise", {})
    k = math.floor(float(spot.get("density", 0.0)) * n)
    if k > 0:
        out.reshape(-1)[uniform_indices(substream_seed(seed, 0x73706F74), k, n)] = int(
            spot.get("intensity", 255))
    return out
