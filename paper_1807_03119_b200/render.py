"""First-hit surface ray caster with the ray-time noise filters, on the B200.

Drop-in for render.py of the reference (render.py:31-565).  Host code keeps
the camera / parameter dataclasses and computes the handful of FP64 camera
constants with numpy exactly as the reference does (Camera.basis,
render.py:49-62); everything per pixel runs in one CUDA kernel (K4,
csrc/vx_render.cu): FP64 ray setup, exact FP32 march with empty-space
skipping, the configured filter at every surface candidate, 3D Sobel normal,
Phong shading, quantisation and the fused image histogram.

Frames are bit-identical to the reference's for any ``workers`` (the
argument is accepted and ignored; the device has no bands).  ``filter_fn``
overrides cannot run on the device and raise ``RenderError``: there is no
CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import threading
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .filters import FilterConfig, FilterKind, native_config
from .histogram import HistogramModel
from .volume import Volume, device_volume

_PAD = 16  # chunk clip bound of render.py:286 (grid.py:19 PAD = 16)
_STEP_CHUNK = 16


class RenderError(Exception):
    pass


@dataclass(frozen=True)
class Camera:
    """Pinhole camera in voxel coordinates (render.py:35-79)."""

    position: tuple[float, float, float]
    look_at: tuple[float, float, float]
    up: tuple[float, float, float] = (0.0, 0.0, 1.0)
    fov_y_deg: float = 45.0

    def __post_init__(self):
        if not 0.0 < self.fov_y_deg < 180.0:
            raise RenderError(f"fov must be in (0, 180), got {self.fov_y_deg}")
        # validated and kept: a moving camera is a new Camera per frame, and
        # ray_setup would otherwise recompute the basis (numpy, ~15 us)
        object.__setattr__(self, "_basis", self._compute_basis())

    def basis(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Orthonormal (right, up, forward), numpy FP64 (render.py:49-62)."""
        right, up, fwd = self.__dict__["_basis"]
        return right.copy(), up.copy(), fwd.copy()

    def _compute_basis(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        pos = np.asarray(self.position, dtype=np.float64)
        fwd = np.asarray(self.look_at, dtype=np.float64) - pos
        norm = np.linalg.norm(fwd)
        if norm == 0:
            raise RenderError("camera position and look_at coincide")
        fwd = fwd / norm
        right = np.cross(fwd, np.asarray(self.up, dtype=np.float64))
        rnorm = np.linalg.norm(right)
        if rnorm < 1e-9:
            raise RenderError("camera up vector is parallel to the view direction")
        right = right / rnorm
        return right, np.cross(right, fwd), fwd

    def to_json(self) -> dict:
        return {"position": list(self.position), "look_at": list(self.look_at),
                "up": list(self.up), "fov_y_deg": self.fov_y_deg}

    @classmethod
    def from_json(cls, obj: dict) -> "Camera":
        return cls(position=tuple(float(v) for v in obj["position"]),
                   look_at=tuple(float(v) for v in obj["look_at"]),
                   up=tuple(float(v) for v in obj.get("up", (0, 0, 1))),
                   fov_y_deg=float(obj.get("fov_y_deg", 45.0)))


def orbit_camera(volume: Volume, azimuth_deg: float = 45.0, elevation_deg: float = 25.0,
                 distance: float | None = None, fov_y_deg: float = 45.0) -> Camera:
    """Camera on an orbit around the volume centre, z up (render.py:82-105)."""
    nx, ny, nz = volume.dims
    target = ((nx - 1) / 2.0, (ny - 1) / 2.0, (nz - 1) / 2.0)
    if distance is None:
        distance = 2.2 * math.sqrt(nx * nx + ny * ny + nz * nz) / 2.0
    el = math.radians(max(-89.0, min(89.0, elevation_deg)))
    az = math.radians(azimuth_deg)
    pos = (target[0] + distance * math.cos(el) * math.cos(az),
           target[1] + distance * math.cos(el) * math.sin(az),
           target[2] + distance * math.sin(el))
    return Camera(position=pos, look_at=target, fov_y_deg=fov_y_deg)


@dataclass(frozen=True)
class RenderParams:
    """Image, march and shading parameters (render.py:108-150)."""

    width: int = 512
    height: int = 512
    step_size: float = 0.5
    max_steps: int = 0
    ambient: float = 0.1
    diffuse: float = 0.7
    specular: float = 0.2
    shininess: float = 16.0
    light_direction: tuple[float, float, float] = (1.0, -1.0, 1.5)
    background: int = 0

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise RenderError(f"image size must be >= 1x1, got {self.width}x{self.height}")
        if self.step_size <= 0:
            raise RenderError(f"step_size must be > 0, got {self.step_size}")
        if min(self.ambient, self.diffuse, self.specular) < 0:
            raise RenderError("lighting coefficients must be >= 0")
        if not 0 <= self.background <= 255:
            raise RenderError(f"background must be in [0, 255], got {self.background}")

    def to_json(self) -> dict:
        return {"width": self.width, "height": self.height, "step_size": self.step_size,
                "max_steps": self.max_steps, "ambient": self.ambient, "diffuse": self.diffuse,
                "specular": self.specular, "shininess": self.shininess,
                "light_direction": list(self.light_direction), "background": self.background}

    @classmethod
    def from_json(cls, obj: dict) -> "RenderParams":
        kwargs = dict(obj)
        if "light_direction" in kwargs:
            kwargs["light_direction"] = tuple(kwargs["light_direction"])
        return cls(**kwargs)


@dataclass
class Frame:
    """Rendered image plus timing and the state that produced it (render.py:153-174)."""

    pixels: np.ndarray
    timing: dict
    filter_config: FilterConfig
    render_params: RenderParams
    camera: Camera
    volume_hash: str
    hit_count: int = 0

    def meta_json(self) -> dict:
        return {"image": {"width": int(self.pixels.shape[1]), "height": int(self.pixels.shape[0])},
                "timing": self.timing, "filter_config": self.filter_config.to_json(),
                "render_params": self.render_params.to_json(), "camera": self.camera.to_json(),
                "volume_hash": self.volume_hash, "hit_count": self.hit_count}


@dataclass(frozen=True)
class Hit:
    position: tuple[float, float, float]
    voxel: tuple[int, int, int]
    value: float
    t: float


# --- native structs ----------------------------------------------------------------


def ray_setup(camera: Camera, width: int, height: int) -> _lib.vx_ray_setup:
    """Host FP64 constants of primary_ray_dirs (render.py:190-192)."""
    right, up, fwd = camera.__dict__["_basis"]
    rs = _lib.vx_ray_setup()
    # right, up, fwd, origin, tan_f, aspect: 14 contiguous doubles
    d = np.frombuffer(rs, dtype=np.float64, count=14)
    d[0:3], d[3:6], d[6:9] = right, up, fwd
    d[9:12] = camera.position
    d[12] = math.tan(math.radians(camera.fov_y_deg) / 2.0)
    d[13] = width / height
    rs.width = width
    rs.height = height
    return rs


def chunk_for(step: float) -> tuple[int, bool]:
    """Samples per march pass and the clip flag (render.py:286-287)."""
    chunk = max(1, min(_STEP_CHUNK, int((_PAD - 1) / step))) if step < _PAD - 1 else 1
    return chunk, chunk * step > _PAD - 1


def native_params(params: RenderParams, *, max_steps: int | None = None,
                  skip: bool = True) -> _lib.vx_render_params:
    rp = _lib.vx_render_params()
    rp.step_size = float(params.step_size)
    rp.max_steps = int(params.max_steps if max_steps is None else max_steps)
    chunk, clip = chunk_for(params.step_size)
    rp.chunk = chunk
    rp.need_clip = 1 if clip else 0
    rp.skip = 1 if skip else 0
    rp.ambient = float(params.ambient)
    rp.diffuse = float(params.diffuse)
    rp.specular = float(params.specular)
    rp.shininess = float(params.shininess)
    light = np.asarray(params.light_direction, dtype=np.float64)
    light = light / np.linalg.norm(light)  # render.py:512-513
    for i in range(3):
        rp.light[i] = float(light[i])
    rp.background = int(params.background)
    return rp


# --- ray setup helpers (render.py:188-230) -------------------------------------------


def primary_ray_dirs(camera: Camera, width: int, height: int) -> np.ndarray:
    """(height*width, 3) unit directions, row-major from the top-left (device)."""
    _lib.require_device()
    rs = ray_setup(camera, width, height)
    out = np.empty((width * height, 3), dtype=np.float64)
    _lib.call("vx_ray_dirs", C.byref(rs), _lib.ptr(out), exc_type=RenderError)
    return out


def ray_box_spans(origin: np.ndarray, dirs: np.ndarray, dims) -> tuple[np.ndarray, np.ndarray]:
    """Entry/exit distances against [-0.5, n-0.5]^3 (device)."""
    _lib.require_device()
    o = np.ascontiguousarray(np.asarray(origin, dtype=np.float64).reshape(3))
    d = np.ascontiguousarray(np.asarray(dirs, dtype=np.float64).reshape(-1, 3))
    dm = np.asarray([int(v) for v in dims], dtype=np.int64)
    te = np.empty(d.shape[0], dtype=np.float64)
    tx = np.empty(d.shape[0], dtype=np.float64)
    _lib.call("vx_ray_spans", _lib.ptr(o), _lib.ptr(d), d.shape[0], _lib.ptr(dm), _lib.ptr(te),
              _lib.ptr(tx), exc_type=RenderError)
    return te, tx


# --- normals and shading (render.py:344-413) ------------------------------------------


def sobel_normal_batch(volume: Volume, vx, vy, vz, fallback: np.ndarray) -> np.ndarray:
    """(n, 3) unit normals toward decreasing density (device)."""
    xs = np.ascontiguousarray(np.asarray(vx, dtype=np.int64).reshape(-1))
    ys = np.ascontiguousarray(np.asarray(vy, dtype=np.int64).reshape(-1))
    zs = np.ascontiguousarray(np.asarray(vz, dtype=np.int64).reshape(-1))
    fb = np.ascontiguousarray(np.asarray(fallback, dtype=np.float64).reshape(-1, 3))
    out = np.empty((xs.size, 3), dtype=np.float64)
    if xs.size:
        dev = device_volume(volume)
        _lib.call("vx_sobel_batch", dev.handle, _lib.ptr(xs), _lib.ptr(ys), _lib.ptr(zs), xs.size,
                  _lib.ptr(fb), _lib.ptr(out), exc_type=RenderError)
    return out


def sobel_normal(volume: Volume, x: int, y: int, z: int, fallback=(0.0, 0.0, 1.0)) -> np.ndarray:
    fb = np.asarray(fallback, dtype=np.float64).reshape(1, 3)
    return sobel_normal_batch(volume, [x], [y], [z], fb)[0]


def shade_phong_batch(normals: np.ndarray, view_dirs: np.ndarray, light_dir: np.ndarray,
                      params: RenderParams) -> np.ndarray:
    """Grey values in [0, 255] (device)."""
    _lib.require_device()
    nn = np.ascontiguousarray(np.asarray(normals, dtype=np.float64).reshape(-1, 3))
    vv = np.ascontiguousarray(np.asarray(view_dirs, dtype=np.float64).reshape(-1, 3))
    rp = native_params(params)
    light = np.asarray(light_dir, dtype=np.float64).reshape(3)
    for i in range(3):
        rp.light[i] = float(light[i])
    out = np.empty(nn.shape[0], dtype=np.uint8)
    if nn.shape[0]:
        _lib.call("vx_phong_batch", _lib.ptr(nn), _lib.ptr(vv), nn.shape[0], C.byref(rp),
                  _lib.ptr(out), exc_type=RenderError)
    return out


def shade_phong(normal, view_dir, light_dir, params: RenderParams) -> int:
    return int(shade_phong_batch(np.asarray(normal, dtype=np.float64).reshape(1, 3),
                                 np.asarray(view_dir, dtype=np.float64).reshape(1, 3),
                                 np.asarray(light_dir, dtype=np.float64), params)[0])


# --- march_ray (render.py:426-464) -------------------------------------------------------


def march_rays(volume: Volume, origins, directions, config: FilterConfig,
               histogram: HistogramModel | None = None, step_size: float = 0.5,
               max_steps=0):
    """Batch form of march_ray: arbitrary origins and (normalised) directions."""
    config = config.resolve_threshold(histogram)
    o = np.ascontiguousarray(np.asarray(origins, dtype=np.float64).reshape(-1, 3))
    d = np.ascontiguousarray(np.asarray(directions, dtype=np.float64).reshape(-1, 3))
    n = d.shape[0]
    te = np.empty(n)
    tx = np.empty(n)
    for i in range(n):  # spans per origin (device)
        a, b = ray_box_spans(o[i], d[i:i + 1], volume.dims)
        te[i], tx[i] = a[0], b[0]
    ms = np.empty(n, dtype=np.int32)
    given = np.broadcast_to(np.asarray(max_steps, dtype=np.int64), (n,))
    for i in range(n):
        if given[i] <= 0:
            span = float(tx[i] - te[i])
            ms[i] = max(1, math.ceil(span / step_size) + 1) if span >= 0 else 1
        else:
            ms[i] = int(given[i])
    rp = native_params(RenderParams(step_size=step_size))
    fc = native_config(config, histogram)
    hit = np.zeros(n, dtype=np.uint8)
    vox = np.zeros((n, 3), dtype=np.int32)
    t = np.zeros(n, dtype=np.float32)
    val = np.zeros(n, dtype=np.float64)
    dev = device_volume(volume)
    _lib.call("vx_march_rays", dev.handle, _lib.ptr(o), _lib.ptr(d), _lib.ptr(te), _lib.ptr(tx),
              _lib.ptr(ms), n, C.byref(rp), C.byref(fc), _lib.ptr(hit), _lib.ptr(vox), _lib.ptr(t),
              _lib.ptr(val), exc_type=RenderError)
    return hit.astype(bool), vox.astype(np.int64), t.astype(np.float64), val


def march_ray(volume: Volume, origin, direction, config: FilterConfig,
              histogram: HistogramModel | None = None, step_size: float = 0.5,
              max_steps: int = 0) -> Hit | None:
    """March a single ray; None when it leaves the volume unaccepted."""
    origin = np.asarray(origin, dtype=np.float64)
    direction = np.asarray(direction, dtype=np.float64)
    direction = direction / np.linalg.norm(direction)
    hit, vox, t, val = march_rays(volume, origin.reshape(1, 3), direction.reshape(1, 3), config,
                                  histogram, step_size, max_steps)
    if not hit[0]:
        return None
    pos = origin + t[0] * direction
    return Hit(position=tuple(float(v) for v in pos), voxel=tuple(int(v) for v in vox[0]),
               value=float(val[0]), t=float(t[0]))


# --- frames (render.py:488-560) -------------------------------------------------------------


@dataclass
class FrameDetail:
    """Per-pixel diagnostics of one device frame (parity tests, bench)."""

    pixels: np.ndarray
    hit_voxel: np.ndarray | None
    hit_t: np.ndarray | None
    hit_value: np.ndarray | None
    intensity: np.ndarray | None
    image_hist: np.ndarray
    hit_count: int
    samples: int
    diag: dict | None = None
    device_ms: float | None = None  # CUDA-event K4 time (frame_timing() on)


_resolved: dict = {}  # (id(config), id(histogram)) -> (config, histogram, resolved)


def _check_render_args(config: FilterConfig, histogram, filter_fn) -> FilterConfig:
    if config.threshold is None:
        # an auto-threshold config resolves to the same FilterConfig every
        # frame: reuse it (the struct caches below key on its identity)
        hit = _resolved.get((id(config), id(histogram)))
        if hit is not None and hit[0] is config and hit[1] is histogram:
            config = hit[2]
        else:
            resolved = config.resolve_threshold(histogram)
            if len(_resolved) > 64:
                _resolved.clear()
            _resolved[(id(config), id(histogram))] = (config, histogram, resolved)
            config = resolved
    if config.kind in (FilterKind.SIGMA, FilterKind.ENTROPY) and histogram is None:
        raise RenderError(f"{config.kind.value} filter needs the volume histogram")
    if filter_fn is not None:
        raise RenderError("filter_fn overrides are not supported: filters run inside the B200 "
                          "ray-cast kernel (no CPU fallback)")
    return config


class _StructCache:
    """Small LRU of the packed C structs of (camera, params, config+histogram):
    an interactive viewer re-renders with mostly unchanged state."""

    def __init__(self, size: int = 32):
        from collections import OrderedDict

        self.size = size
        self.d: OrderedDict = OrderedDict()
        self.lock = threading.Lock()  # render_frame runs on executor threads

    def get(self, key, make):
        try:
            with self.lock:
                v = self.d.pop(key, None)
        except TypeError:  # unhashable key part
            return make()
        if v is None:
            v = make()
        with self.lock:
            self.d[key] = v
            while len(self.d) > self.size:
                self.d.popitem(last=False)
        return v


_structs = _StructCache()


_last_native = None  # identity fast path: an interactive loop re-renders with the same objects


def _native(camera, params, config, histogram, skip):
    global _last_native
    last = _last_native
    if (last is not None and last[0] is camera and last[1] is params and last[2] is config
            and last[3] is histogram and last[4] == skip):
        return last[5]
    W, H = params.width, params.height
    rs = _structs.get(("rs", camera, W, H), lambda: ray_setup(camera, W, H))
    rp = _structs.get(("rp", params, skip), lambda: native_params(params, skip=skip))
    # the histogram object is kept in the value so its id cannot be reused
    fc = _structs.get(("fc", config, id(histogram)),
                      lambda: (native_config(config, histogram), histogram))[0]
    _last_native = (camera, params, config, histogram, skip, (rs, rp, fc),
                    (C.byref(rs), C.byref(rp), C.byref(fc)))
    return rs, rp, fc


def _native_refs(camera, params, config, histogram, skip):
    """byref()s of _native's structs (kept with the identity fast path)."""
    _native(camera, params, config, histogram, skip)
    return _last_native[6]


def render_detail(volume: Volume, camera: Camera, params: RenderParams, config: FilterConfig,
                  histogram: HistogramModel | None = None, *, diagnostics: bool = False,
                  skip: bool = True, partition: tuple[int, int] | None = None,
                  _checked: bool = False) -> FrameDetail:
    if not _checked:
        config = _check_render_args(config, histogram, None)
    _lib.require_device()
    dev = device_volume(volume)
    rs, rp, fc = _native(camera, params, config, histogram, skip)
    npx = params.width * params.height
    # page-locked frame and counters (image histogram [0:256], hit count
    # [256], samples [257], diag [258:266]): the device writes them by DMA
    pixels, small, pix_ptr, sp = _lib.pinned.frame(params.height, params.width)
    vox = t = val = inten = None
    if not diagnostics and partition is None:
        # the frame pool recycles its buffers: their output structs are kept
        # (ctypes field writes cost ~0.5 us each)
        ent = _outs.get(pix_ptr)
        if ent is None or ent[0] != sp:
            out = _lib.vx_render_out()
            out.pixels = pix_ptr
            out.image_hist = sp
            out.hit_count = sp + 256 * 8
            out.samples = sp + 257 * 8
            if len(_outs) > 64:
                _outs.clear()
            ent = _outs[pix_ptr] = (sp, out, C.byref(out))
        rsr, rpr, fcr = _native_refs(camera, params, config, histogram, skip)
        rc = _vx_render()(dev.handle, rsr, rpr, fcr, None, ent[2])
        if rc:
            _lib.check(rc, RenderError)
        return _finish(pixels, small, diagnostics, vox, t, val, inten)
    out = _lib.vx_render_out()
    out.pixels = pix_ptr
    out.image_hist = sp
    out.hit_count = sp + 256 * 8
    out.samples = sp + 257 * 8
    if diagnostics:
        out.diag = sp + 258 * 8
        vox = np.empty((npx, 3), dtype=np.int32)
        t = np.empty(npx, dtype=np.float32)
        val = np.empty(npx, dtype=np.float64)
        inten = np.empty(npx, dtype=np.float64)
        out.hit_voxel = vox.ctypes.data
        out.hit_t = t.ctypes.data
        out.hit_value = val.ctypes.data
        out.intensity = inten.ctypes.data
    part = None
    if partition is not None:
        part = _lib.vx_partition(int(partition[0]), int(partition[1]))
    _lib.call("vx_render", dev.handle, C.byref(rs), C.byref(rp), C.byref(fc),
              C.byref(part) if part is not None else None, C.byref(out), exc_type=RenderError)
    return _finish(pixels, small, diagnostics, vox, t, val, inten)


def _finish(pixels, small, diagnostics, vox, t, val, inten) -> FrameDetail:
    device_ms = None
    if getattr(_timing, "on", False):
        ms = C.c_float(-1.0)
        _lib.call("vx_last_render_ms", C.byref(ms))
        device_ms = ms.value if ms.value >= 0.0 else None
    return FrameDetail(device_ms=device_ms, pixels=pixels, hit_voxel=vox, hit_t=t,
                       hit_value=val, intensity=inten, image_hist=small[:256],
                       hit_count=int(small[256]), samples=int(small[257]),
                       diag=dict(zip(_DIAG_NAMES, (int(v) for v in small[258:266])))
                       if diagnostics else None)


_outs: dict = {}  # pinned frame address -> (counters address, vx_render_out, its byref)
_vx_render_fn = None


def _vx_render():
    global _vx_render_fn
    if _vx_render_fn is None:
        _vx_render_fn = _lib.load().vx_render
    return _vx_render_fn


_DIAG_NAMES = ("lookups", "skips", "chunks_skipped", "unused", "sample_groups",
               "filter_evals", "hits", "iterations")
_timing = threading.local()  # frame_timing() state of this thread (mirrors the C side)


class frame_timing:
    """Context manager: CUDA-event device times in Frame.timing for frames
    rendered by this thread inside the block (run_timing_benchmark)."""

    def __enter__(self):
        _lib.call("vx_set_frame_timing", 1)
        _timing.on = True
        return self

    def __exit__(self, *exc):
        _lib.call("vx_set_frame_timing", 0)
        _timing.on = False
        return False


def render_frame(volume: Volume, camera: Camera, params: RenderParams, config: FilterConfig,
                 histogram: HistogramModel | None = None, workers: int = 1,
                 filter_fn=None, devices=None) -> Frame:
    """Render one frame on the B200; bit-identical output for any worker count.

    ``devices`` (or env VOXB200_DEVICES="0,1,..."): split the frame over
    these GPUs from this process (vx_init + vx_multi_render,
    a replica per device, tiles dealt round-robin, peer stores into the first
    device's frame).  The pixels do not depend on it, as they do not depend
    on ``workers`` (render.py:514-541).
    """
    wall0 = time.perf_counter()
    config = _check_render_args(config, histogram, filter_fn)
    devs = _devices(devices)
    if devs is not None and len(devs) > 1:
        d = _render_multi(volume, camera, params, config, histogram, devs)
    else:
        d = render_detail(volume, camera, params, config, histogram, _checked=True)
    total_ms = (time.perf_counter() - wall0) * 1000.0
    frame = Frame(
        pixels=d.pixels,
        # march, filter and shading are one fused kernel: under frame_timing()
        # its CUDA-event time is march_ms and device_ms (shade_ms 0); without
        # it march_ms is the wall clock as before
        timing={"total_ms": total_ms,
                "march_ms": total_ms if d.device_ms is None else d.device_ms,
                "shade_ms": 0.0, "device_ms": d.device_ms},
        filter_config=config,
        render_params=params,
        camera=camera,
        volume_hash=volume.content_hash(),
        hit_count=d.hit_count,
    )
    frame.image_hist = d.image_hist
    return frame


# --- one process, several GPUs (vx_init / vx_multi_*) ----------------------------------


_env_devices: list = []  # VOXB200_DEVICES, read once: [value]


def _devices(devices):
    if devices is None:
        if not _env_devices:
            env = os.environ.get("VOXB200_DEVICES")
            _env_devices.append(tuple(int(v) for v in env.split(",") if v.strip()) if env else None)
        return _env_devices[0]
    return tuple(int(v) for v in devices)


class MultiVolume:
    """Owning handle of a vx_multi (a replica on each listed device)."""

    def __init__(self, volume: Volume, devices: tuple):
        _lib.require_device()
        ids = (C.c_int * len(devices))(*devices)
        _lib.call("vx_init", len(devices), ids, exc_type=RenderError)
        self.handle = C.c_void_p()
        data = np.ascontiguousarray(volume.data)
        _lib.call("vx_multi_volume_create_u8", _lib.ptr(data), *volume.dims, C.byref(self.handle),
                  exc_type=RenderError)
        self.devices = devices
        self._finalizer = weakref.finalize(self, MultiVolume._release, self.handle.value)

    @staticmethod
    def _release(raw):
        if raw:
            try:
                _lib.load().vx_multi_destroy(C.c_void_p(raw))
            except Exception:
                pass

    def histogram_counts(self) -> np.ndarray:
        out = np.zeros(256, dtype=np.uint64)
        _lib.call("vx_multi_histogram", self.handle, _lib.ptr(out))
        return out.astype(np.int64)


_multi_lock = threading.Lock()


def multi_volume(volume: Volume, devices) -> MultiVolume:
    """The volume's replicas on ``devices``, built on first use and cached."""
    devices = tuple(int(v) for v in devices)
    cache = volume.__dict__.get("_vx_multi")
    if cache is None or cache.devices != devices:
        with _multi_lock:
            cache = volume.__dict__.get("_vx_multi")
            if cache is None or cache.devices != devices:
                cache = MultiVolume(volume, devices)
                object.__setattr__(volume, "_vx_multi", cache)
    return cache


def _render_multi(volume, camera, params, config, histogram, devices) -> FrameDetail:
    mv = multi_volume(volume, devices)
    rs, rp, fc = _native(camera, params, config, histogram, True)
    pixels, small, pix_ptr, sp = _lib.pinned.frame(params.height, params.width)
    out = _lib.vx_render_out()
    out.pixels = pix_ptr
    out.image_hist = sp
    out.hit_count = sp + 256 * 8
    out.samples = sp + 257 * 8
    with _multi_lock:  # vx_init's device list is process-wide
        _lib.call("vx_multi_render", mv.handle, C.byref(rs), C.byref(rp), C.byref(fc),
                  C.byref(out), exc_type=RenderError)
    return FrameDetail(pixels=pixels, hit_voxel=None, hit_t=None, hit_value=None, intensity=None,
                       image_hist=small[:256], hit_count=int(small[256]),
                       samples=int(small[257]))
