"""ctypes binding of libvoxb200.so (include/voxb200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every compute entry point raises ``NativeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import threading
import weakref
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("VOXB200_LIB", str(_PKG / "libvoxb200.so")))

VX_OK, VX_EINVAL, VX_ENOMEM, VX_ECUDA, VX_ERANGE = 0, 1, 2, 3, 5

# filters.py:43-57 order
KIND_CODES = {
    "none": 0,
    "mean": 1,
    "sigma": 2,
    "okada": 3,
    "entropy": 4,
    "local-cluster": 5,
}


class NativeError(RuntimeError):
    """The CUDA library failed (or is unavailable)."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class vx_ray_setup(C.Structure):
    _fields_ = [
        ("right", C.c_double * 3),
        ("up", C.c_double * 3),
        ("fwd", C.c_double * 3),
        ("origin", C.c_double * 3),
        ("tan_f", C.c_double),
        ("aspect", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]


class vx_render_params(C.Structure):
    _fields_ = [
        ("step_size", C.c_double),
        ("max_steps", C.c_int32),
        ("chunk", C.c_int32),
        ("need_clip", C.c_int32),
        ("skip", C.c_int32),
        ("ambient", C.c_double),
        ("diffuse", C.c_double),
        ("specular", C.c_double),
        ("shininess", C.c_double),
        ("light", C.c_double * 3),
        ("background", C.c_int32),
        ("_pad", C.c_int32),
    ]


class vx_filter_config(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("kernel_size", C.c_int32),
        ("cluster_offset", C.c_int32),
        ("entropy_pairwise", C.c_int32),
        ("threshold", C.c_double),
        ("sigma_band", C.c_double),
        ("okada_threshold", C.c_double),
        ("entropy_threshold", C.c_double),
        ("entropy_lut", C.c_double * 256),
    ]


class vx_partition(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32)]


class vx_render_out(C.Structure):
    _fields_ = [
        ("pixels", C.c_void_p),
        ("hit_voxel", C.c_void_p),
        ("hit_t", C.c_void_p),
        ("hit_value", C.c_void_p),
        ("intensity", C.c_void_p),
        ("image_hist", C.c_void_p),
        ("hit_count", C.c_void_p),
        ("samples", C.c_void_p),
        ("diag", C.c_void_p),
        ("trunc_flag", C.c_void_p),
    ]


class vx_group_frame(C.Structure):
    _fields_ = [
        ("pixels", C.c_void_p),
        ("counters", C.c_void_p),
        ("frame", C.c_uint32),
        ("_pad", C.c_uint32),
    ]


VX_GROUP_BLOB_BYTES = 256
VX_GROUP_SYNC_AUTO, VX_GROUP_SYNC_DEVICE, VX_GROUP_SYNC_HOST = -1, 0, 1

P = C.c_void_p
I32, I64, U64, F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double

# name -> argtypes (all return int unless listed in _RESTYPES)
SIGNATURES = {
    "vx_last_error": [],
    "vx_version": [],
    "vx_device_count": [P],
    "vx_set_device": [C.c_int],
    "vx_synchronize": [],
    "vx_volume_create_u8": [P, I64, I64, I64, P],
    "vx_volume_create_u16": [P, I64, I64, I64, P],
    "vx_volume_create_device_u8": [P, I64, I64, I64, P],
    "vx_volume_load_raw": [C.c_char_p, I64, I64, I64, C.c_int32, P, P],
    "vx_volume_load_slices": [P, P, I64, I64, I64, P, P],
    "vx_volume_destroy": [P],
    "vx_volume_dims": [P, P],
    "vx_volume_read": [P, P],
    "vx_volume_device_bytes": [P, P],
    "vx_volume_skip_cap": [P, C.c_int32, P],
    "vx_histogram": [P, P],
    "vx_histogram_host": [P, U64, P],
    "vx_histogram_device": [P, U64, P, P],
    "vx_otsu": [P, P],
    "vx_otsu_device": [P, P, P],
    "vx_histogram_otsu_device": [P, U64, P, P, P],
    "vx_image_entropy": [P, I64, P, P],
    "vx_entropy_from_counts_device": [P, U64, P, P],
    "vx_render": [P, P, P, P, P, P],
    "vx_render_device": [P, P, P, P, P, P, P],
    "vx_march_rays": [P, P, P, P, P, P, I64, P, P, P, P, P, P],
    "vx_ray_dirs": [P, P],
    "vx_ray_spans": [P, P, I64, P, P, P],
    "vx_filter_batch": [P, P, P, P, I64, P, P],
    "vx_sobel_batch": [P, P, P, P, I64, P, P],
    "vx_phong_batch": [P, P, I64, P, P],
    "vx_volume_create_phantom": [I64, I64, I64, P, I64, F64, U64, P, I64, I32, P],
    "vx_phantom_device": [P, I64, I64, I64, P, I64, F64, U64, P, I64, I32, P],
    "vx_launch_counter": [P, C.c_int],
    "vx_last_render_ms": [P],
    "vx_set_frame_timing": [C.c_int],
    "vx_set_schedule": [C.c_int32, C.c_int32, C.c_int32, C.c_int32],
    "vx_host_alloc": [U64, P],
    "vx_host_free": [P],
    "vx_volume_distance_map": [P, I32, I32, P, P],
    "vx_volume_histogram_slab": [P, I64, I64, P, P],
    "vx_u16_dither_device": [P, U64, U64, U64, P, P],
    "vx_group_create": [I32, I32, I64, P, P],
    "vx_group_connect": [P, P, I32],
    "vx_group_info": [P, P, P],
    "vx_group_probe_device_sync": [],
    "vx_group_render": [P, P, P, P, P, P, P],
    "vx_group_release": [P, P],
    "vx_group_download": [P, P, P, I64, P],
    "vx_group_destroy": [P],
    "vx_init": [C.c_int, P],
    "vx_multi_volume_create_u8": [P, I64, I64, I64, P],
    "vx_multi_render": [P, P, P, P, P],
    "vx_multi_histogram": [P, P],
    "vx_multi_info": [P, P, P],
    "vx_multi_destroy": [P],
}
_RESTYPES = {"vx_last_error": C.c_char_p}

_lib = None
_lock = threading.Lock()


def load():
    """Load (building first if the sources are newer) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if os.environ.get("VOXB200_NO_BUILD") != "1":
            try:
                from . import _build

                if _build.needs_build():
                    _build.build()
            except Exception as exc:  # nvcc missing on a prebuilt box is fine
                if not LIB_PATH.exists():
                    raise NativeError(VX_ECUDA, f"libvoxb200.so unavailable: {exc}") from exc
        if not LIB_PATH.exists():
            raise NativeError(VX_ECUDA, f"libvoxb200.so not found at {LIB_PATH}")
        lib = C.CDLL(str(LIB_PATH))
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().vx_last_error()
    return msg.decode() if msg else ""


def check(rc: int, exc_type=None):
    """Raise on a non-zero status; EINVAL maps to the caller's error type."""
    if rc == VX_OK:
        return
    msg = last_error()
    if rc == VX_EINVAL and exc_type is not None:
        raise exc_type(msg)
    raise NativeError(rc, msg)


_fns: dict = {}


def call(name: str, *args, exc_type=None):
    fn = _fns.get(name)
    if fn is None:
        fn = _fns[name] = getattr(load(), name)
    rc = fn(*args)
    if rc != VX_OK:
        check(rc, exc_type)


_device_ok = None


def require_device():
    """Fail loudly when no CUDA device is visible (no CPU fallback)."""
    global _device_ok
    if _device_ok:
        return
    n = C.c_int(0)
    rc = load().vx_device_count(C.byref(n))
    if rc != VX_OK or n.value < 1:
        raise NativeError(VX_ECUDA, "no CUDA device visible: the B200 path has no CPU fallback "
                          f"({last_error() or 'cudaGetDeviceCount returned 0'})")
    _device_ok = True


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


def launches(reset: bool = False) -> int:
    n = C.c_uint64(0)
    call("vx_launch_counter", C.byref(n), 1 if reset else 0)
    return int(n.value)


class PinnedPool:
    """Reusable page-locked host buffers for frame outputs (DMA straight into
    the numpy arrays the caller receives; cudaHostAlloc is too slow per frame).
    A buffer returns to the pool when the last array viewing it is freed."""

    ARENA_BYTES = 16 << 20  # two 2048^2 frames with counters, or many smaller ones
    MAX_FRAME_SIZES = 8  # frame-size entries kept (LRU); older sizes are dropped
    FREE_CAP = 64 << 20  # page-locked bytes parked for reuse beyond the arena

    def __init__(self):
        from collections import OrderedDict

        self._free: dict[int, list[int]] = {}
        self._free_bytes = 0
        self._frames: OrderedDict = OrderedDict()
        # re-entrant: buffer finalizers (_release) can run inside a locked
        # region when dropping an entry frees the last reference
        self._lock = threading.RLock()
        self._arena = 0  # page-locked block new buffers are carved from
        self._arena_left = 0

    def prewarm(self) -> None:
        """Allocate the page-locked arena now (called when a device volume is
        created): the first frame then carves its buffers instead of paying
        cudaHostAlloc, whose cost (1-25 ms measured) depends on the host."""
        with self._lock:
            if self._arena:
                return
        p = C.c_void_p()
        call("vx_host_alloc", self.ARENA_BYTES, C.byref(p))
        with self._lock:
            if self._arena:  # another thread won: keep theirs, park ours as a buffer
                self._free.setdefault(self.ARENA_BYTES, []).append(p.value)
                return
            self._arena, self._arena_left = p.value, self.ARENA_BYTES

    def _carve(self, nbytes: int) -> int | None:
        """A fresh buffer from the arena (256-byte aligned), or None."""
        need = (max(nbytes, 1) + 255) & ~255
        with self._lock:
            if not self._arena or need > self._arena_left:
                return None
            ptr = self._arena + (self.ARENA_BYTES - self._arena_left)
            self._arena_left -= need
            return ptr

    def array(self, shape, dtype) -> np.ndarray:
        return self.array_ptr(shape, dtype)[0]

    def array_ptr(self, shape, dtype) -> tuple[np.ndarray, int]:
        """(array, its host address)."""
        dtype = np.dtype(dtype)
        count = 1
        for n in shape:
            count *= int(n)
        nbytes = count * dtype.itemsize
        with self._lock:
            lst = self._free.get(nbytes)
            ptr = lst.pop() if lst else None
            if ptr is not None and not self._in_arena(ptr):
                self._free_bytes -= nbytes
        if ptr is None:
            ptr = self._carve(nbytes)
        if ptr is None:
            # a miss allocates a spare too: a caller that keeps the previous
            # frame while rendering the next (double buffering) then never
            # pays cudaHostAlloc (~3-5 ms per MiB) inside its loop
            p, spare = C.c_void_p(), C.c_void_p()
            call("vx_host_alloc", nbytes, C.byref(p))
            call("vx_host_alloc", nbytes, C.byref(spare))
            ptr = p.value
            self._release(nbytes, spare.value)
        buf = (C.c_uint8 * max(nbytes, 1)).from_address(ptr)
        weakref.finalize(buf, self._release, nbytes, ptr)
        return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape), ptr

    def _in_arena(self, ptr) -> bool:
        return bool(self._arena) and self._arena <= ptr < self._arena + self.ARENA_BYTES

    def _release(self, nbytes, ptr):
        with self._lock:
            if not self._in_arena(ptr):
                if self._free_bytes + nbytes > self.FREE_CAP:
                    # bounded: a viewer resizing its window does not pin
                    # host memory without limit
                    try:
                        call("vx_host_free", C.c_void_p(ptr))
                    except NativeError:
                        pass
                    return
                self._free_bytes += nbytes
            self._free.setdefault(nbytes, []).append(ptr)

    def frame(self, height: int, width: int) -> tuple[np.ndarray, np.ndarray, int, int]:
        """(pixels (H, W) uint8, counters int64[266], pixels address, counters
        address) in one page-locked buffer, recycled without per-frame ctypes
        or finalizer work: an entry is free again when nothing outside the pool
        references its arrays (views such as ``counters[:256]`` hold a
        reference too)."""
        key = (height, width)
        with self._lock:
            lst = self._frames.setdefault(key, [])
            self._frames.move_to_end(key)
            # LRU over frame sizes: a dropped size's buffers go back to the
            # size-keyed free list (or are freed) when their arrays die
            while len(self._frames) > self.MAX_FRAME_SIZES:
                self._frames.popitem(last=False)
            for ent in lst:
                # free when only the entry references its arrays and its
                # buffer: numpy views of views may point at either the view or
                # the buffer object (base collapsing), so both are counted
                if (sys.getrefcount(ent[0]) == 2 and sys.getrefcount(ent[1]) == 2
                        and sys.getrefcount(ent[4]) == ent[5]
                        and sys.getrefcount(ent[6]) == ent[7]):
                    pix, small = ent[0], ent[1]  # held before the lock is released
                    return pix, small, ent[2], ent[3]
            n_new = 1 if lst else 2  # a spare for double buffering
        npx = height * width
        off = (npx + 63) & ~63
        made = []
        for _ in range(n_new):  # allocated outside the lock (array() takes it)
            raw = self.array((off + 266 * 8,), np.uint8)
            ptr = raw.ctypes.data
            ent = [raw[:npx].reshape(height, width), raw[off:].view(np.int64), ptr, ptr + off,
                   raw.base, 0, raw, 0]
            del raw
            # references of the buffer object and of the flat array while unused
            ent[5], ent[7] = sys.getrefcount(ent[4]), sys.getrefcount(ent[6])
            made.append(ent)
        pix, small, p0, p1 = made[0][:4]
        with self._lock:
            self._frames.setdefault(key, []).extend(made)
        return pix, small, p0, p1


pinned = PinnedPool()
