"""CPU oracle of the voxray hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker / reported CPU baseline; the
product package never does.  It restates the reference
(/root/reference/pkg/src/voxray) in numpy (the 256-element statistics, the
camera constants, image entropy, the exact Otsu scan with Python integers)
and in plain C (liboracle.so, vxoracle.c: the per-voxel / per-ray loops).

Parity pins (see tests/golden/ and oracle/gen_golden.py): this restatement
was checked against the live reference in the build container on every
golden vector the reference's own tests hold for this path, plus frozen
frames of the committed phantoms and the C2 insect phantom.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle.so"
LEVELS = 256
_lib = None


def build() -> Path:
    src = HERE / "vxoracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = C.CDLL(str(LIB))
        _lib.orc_render.restype = C.c_int64
        _lib.orc_max_threads.restype = C.c_int
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


# --- statistics (histogram.py:59-133, metrics.py:26-33) ---------------------------


def hist256(data: np.ndarray) -> np.ndarray:
    """np.bincount(data, minlength=256) (histogram.py:120) in C."""
    a = np.ascontiguousarray(data, dtype=np.uint8).reshape(-1)
    out = np.zeros(LEVELS, dtype=np.uint64)
    lib().orc_hist256(_p(a), C.c_uint64(a.size), _p(out))
    return out.astype(np.int64)


def otsu(counts) -> int:
    """Exact Otsu scan with Python integers (histogram.py:59-101)."""
    c = [int(v) for v in counts]
    total = sum(c)
    b_all = sum(i * v for i, v in enumerate(c))
    a_all = sum(i * i * v for i, v in enumerate(c))
    best_t, best = 0, None
    n0 = b0 = a0 = 0
    for t in range(LEVELS):
        n0 += c[t]
        b0 += t * c[t]
        a0 += t * t * c[t]
        n1, b1, a1 = total - n0, b_all - b0, a_all - a0
        if n0 and n1:
            num, den = (a0 * n0 - b0 * b0) * n1 + (a1 * n1 - b1 * b1) * n0, n0 * n1
        elif n0:
            num, den = a0 * n0 - b0 * b0, n0
        else:
            num, den = a1 * n1 - b1 * b1, n1
        if best is None or num * best[1] < best[0] * den:
            best, best_t = (num, den), t
    return best_t


def sigma_from_counts(counts) -> float:
    """histogram.py:109-116 in the same numpy operation order."""
    c = np.asarray(counts).astype(np.float64)
    n = c.sum()
    idx = np.arange(LEVELS, dtype=np.float64)
    mu = (c * idx).sum() / n
    return float(np.sqrt((c * (idx - mu) ** 2).sum() / n))


def histogram_model(counts) -> dict:
    counts = np.asarray(counts, dtype=np.int64)
    total = int(counts.sum())
    return {"counts": counts, "total": total, "probabilities": counts / total,
            "global_sigma": sigma_from_counts(counts), "otsu": otsu(counts)}


def entropy_terms(p) -> np.ndarray:
    """filters.py:212-218."""
    p = np.asarray(p, dtype=np.float64)
    out = np.zeros_like(p)
    nz = p > 0
    out[nz] = -p[nz] * np.log2(p[nz])
    return out


def image_entropy(pixels) -> float:
    """metrics.py:26-33."""
    px = np.asarray(pixels, dtype=np.uint8).reshape(-1)
    counts = np.bincount(px, minlength=256)
    p = counts[counts > 0] / px.size
    return float(-(p * np.log2(p)).sum())


# --- camera constants (render.py:49-105, 188-192) -----------------------------------


def camera_basis(position, look_at, up=(0.0, 0.0, 1.0)):
    pos = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(look_at, dtype=np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right = right / np.linalg.norm(right)
    return right, np.cross(right, fwd), fwd


def orbit(dims, azimuth_deg=45.0, elevation_deg=25.0, distance=None):
    nx, ny, nz = dims
    target = ((nx - 1) / 2.0, (ny - 1) / 2.0, (nz - 1) / 2.0)
    if distance is None:
        distance = 2.2 * math.sqrt(nx * nx + ny * ny + nz * nz) / 2.0
    el = math.radians(max(-89.0, min(89.0, elevation_deg)))
    az = math.radians(azimuth_deg)
    pos = (target[0] + distance * math.cos(el) * math.cos(az),
           target[1] + distance * math.cos(el) * math.sin(az),
           target[2] + distance * math.sin(el))
    return pos, target


def cam_vector(position, look_at, width, height, fov_y_deg=45.0, up=(0.0, 0.0, 1.0)):
    right, upv, fwd = camera_basis(position, look_at, up)
    tan_f = math.tan(math.radians(fov_y_deg) / 2.0)
    return np.array([*right, *upv, *fwd, *position, tan_f, width / height], dtype=np.float64)


def chunk_for(step: float):
    chunk = max(1, min(16, int(15 / step))) if step < 15 else 1
    return chunk, chunk * step > 15


FILTER_CODES = {"none": 0, "mean": 1, "sigma": 2, "okada": 3, "entropy": 4,
                "local-cluster": 5, "axis": 6}


def ray_dirs(cam: np.ndarray, width: int, height: int) -> np.ndarray:
    out = np.empty((width * height, 3), dtype=np.float64)
    lib().orc_ray_dirs(_p(cam), C.c_int(width), C.c_int(height), _p(out))
    return out


def ray_spans(origin, dirs, dims):
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    dm = np.asarray(dims, dtype=np.int64)
    te = np.empty(d.shape[0])
    tx = np.empty(d.shape[0])
    lib().orc_ray_spans(_p(o), _p(d), C.c_int64(d.shape[0]), _p(dm), _p(te), _p(tx))
    return te, tx


def render(volume: np.ndarray, cam: np.ndarray, width: int, height: int, *, kind="local-cluster",
           threshold: float, kernel_size=3, cluster_offset=1, sigma_band=0.0, okada_threshold=25.0,
           entropy_threshold=2.0, probabilities=None, step=0.5, max_steps=0, ambient=0.1,
           diffuse=0.7, specular=0.2, shininess=16.0, light=(1.0, -1.0, 1.5), background=0,
           row_step=1, threads=1, diagnostics=True) -> dict:
    """render_frame restatement (render.py:488-560) for a (nz, ny, nx) uint8 volume."""
    vol = np.ascontiguousarray(volume, dtype=np.uint8)
    nz, ny, nx = vol.shape
    chunk, clip = chunk_for(step)
    l = np.asarray(light, dtype=np.float64)
    l = l / np.linalg.norm(l)
    prm = np.array([step, max_steps, chunk, 1.0 if clip else 0.0, ambient, diffuse, specular,
                    shininess, l[0], l[1], l[2], background], dtype=np.float64)
    flt = np.array([FILTER_CODES[kind], kernel_size, cluster_offset, threshold, sigma_band,
                    okada_threshold, entropy_threshold], dtype=np.float64)
    lut = entropy_terms(probabilities if probabilities is not None else np.zeros(256))
    npx = width * height
    pixels = np.zeros((height, width), dtype=np.uint8)
    vox = np.full((npx, 3), -1, dtype=np.int32) if diagnostics else None
    ht = np.zeros(npx, dtype=np.float32) if diagnostics else None
    inten = np.full(npx, -1.0) if diagnostics else None
    samples = C.c_int64(0)
    hits = lib().orc_render(_p(vol), C.c_int64(nx), C.c_int64(ny), C.c_int64(nz), _p(cam),
                            C.c_int(width), C.c_int(height), _p(prm), _p(flt), _p(lut),
                            C.c_int(row_step), C.c_int(threads), _p(pixels), _p(vox), _p(ht),
                            _p(inten), C.byref(samples))
    return {"pixels": pixels, "hit_voxel": vox, "hit_t": ht, "intensity": inten,
            "hit_count": int(hits), "samples": int(samples.value)}


def filter_batch(volume: np.ndarray, xs, ys, zs, *, kind, kernel_size=3, cluster_offset=1,
                 sigma_band=0.0, okada_threshold=25.0, entropy_threshold=2.0, probabilities=None,
                 pairwise=None) -> np.ndarray:
    vol = np.ascontiguousarray(volume, dtype=np.uint8)
    nz, ny, nx = vol.shape
    x = np.ascontiguousarray(xs, dtype=np.int64).reshape(-1)
    y = np.ascontiguousarray(ys, dtype=np.int64).reshape(-1)
    z = np.ascontiguousarray(zs, dtype=np.int64).reshape(-1)
    lut = entropy_terms(probabilities if probabilities is not None else np.zeros(256))
    out = np.empty(x.size)
    if pairwise is None:
        pairwise = x.size == 1
    lib().orc_filter_batch(_p(vol), C.c_int64(nx), C.c_int64(ny), C.c_int64(nz), _p(x), _p(y),
                           _p(z), C.c_int64(x.size), C.c_int(FILTER_CODES[kind]),
                           C.c_int(kernel_size), C.c_int(cluster_offset), C.c_double(sigma_band),
                           C.c_double(okada_threshold), C.c_double(entropy_threshold), _p(lut),
                           C.c_int(1 if pairwise else 0), _p(out))
    return out


def sobel_batch(volume, xs, ys, zs, fallback) -> np.ndarray:
    vol = np.ascontiguousarray(volume, dtype=np.uint8)
    nz, ny, nx = vol.shape
    x = np.ascontiguousarray(xs, dtype=np.int64).reshape(-1)
    y = np.ascontiguousarray(ys, dtype=np.int64).reshape(-1)
    z = np.ascontiguousarray(zs, dtype=np.int64).reshape(-1)
    fb = np.ascontiguousarray(fallback, dtype=np.float64).reshape(-1, 3)
    out = np.empty((x.size, 3))
    lib().orc_sobel_batch(_p(vol), C.c_int64(nx), C.c_int64(ny), C.c_int64(nz), _p(x), _p(y),
                          _p(z), C.c_int64(x.size), _p(fb), _p(out))
    return out


def phong_batch(normals, views, light, ambient=0.1, diffuse=0.7, specular=0.2,
                shininess=16.0) -> np.ndarray:
    n = np.ascontiguousarray(normals, dtype=np.float64).reshape(-1, 3)
    v = np.ascontiguousarray(views, dtype=np.float64).reshape(-1, 3)
    l = np.asarray(light, dtype=np.float64)
    sh = np.array([ambient, diffuse, specular, shininess, l[0], l[1], l[2]])
    out = np.empty(n.shape[0], dtype=np.uint8)
    lib().orc_phong_batch(_p(n), _p(v), C.c_int64(n.shape[0]), _p(sh), _p(out))
    return out


def phantom(spec: dict, threads: int = 1) -> np.ndarray:
    """generate_phantom input generator (volume.py:317-368) from spec.to_json() form.

    C with glibc log/cos; numpy's own SIMD log/cos may round differently in
    the last ulp, so bit-identity with the reference's volume is checked by
    content hash in the golden tests rather than assumed.
    """
    from . import rng_np

    nx, ny, nz = (int(v) for v in spec["dims"])
    n = nx * ny * nz
    kinds = {"sphere": 0, "shell": 1, "box": 2}
    shapes = spec.get("shapes", [])
    table = np.zeros((max(1, len(shapes)), 10))
    for i, s in enumerate(shapes):
        table[i] = (kinds[s["kind"]], *s["center"], s["intensity"], s.get("radius", 0.0),
                    s.get("thickness", 0.0), *s.get("extent", (0.0, 0.0, 0.0)))
    sigma = float(spec.get("noise", {}).get("sigma", 0.0))
    seed = rng_np.substream_seed(int(spec.get("rng_seed", 0)), 0x6E6F697365)
    spot = spec.get("spot_noise", {})
    k = math.floor(float(spot.get("density", 0.0)) * n)
    idx = (rng_np.uniform_indices(rng_np.substream_seed(int(spec.get("rng_seed", 0)), 0x73706F74),
                                  k, n) if k > 0 else np.zeros(1, dtype=np.int64))
    out = np.empty((nz, ny, nx), dtype=np.uint8)
    lib().orc_phantom(_p(out), C.c_int64(nx), C.c_int64(ny), C.c_int64(nz), _p(table),
                      C.c_int64(len(shapes)), C.c_double(sigma), C.c_uint64(seed), _p(idx),
                      C.c_int64(k), C.c_int(int(spot.get("intensity", 255))), C.c_int(threads))
    return out


def max_threads() -> int:
    return int(lib().orc_max_threads())
