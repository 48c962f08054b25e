"""Service frame path: render straight into a framed, page-locked message.

Drop-in for the render half of the live service:
``RenderService.render_message`` renders with ``render_frame`` and then packs
``pack_frame(seq, w, h, ms, digest, frame.pixels.tobytes())`` (service.py:
48-53, 168-183), i.e. two full copies of the image on the host.  Here the
device frame is DMA'd by K4's copy-back directly behind the 32-byte "VXSF"
header inside one pinned buffer, and the message is returned as a
memoryview over it (aiohttp's ``send_bytes`` accepts any bytes-like object).
The binary layout is the reference's, byte for byte.
"""

from __future__ import annotations

import ctypes as C
import struct
import time

import numpy as np

from . import _lib
from .filters import FilterConfig
from .histogram import HistogramModel
from .render import Camera, RenderParams, _check_render_args, _native
from .volume import Volume, device_volume

FRAME_MAGIC = b"VXSF"
FRAME_VERSION = 1
FRAME_HEADER = struct.Struct("<4sB3xQHHf8s")  # service.py:38


def pack_frame(sequence: int, width: int, height: int, render_ms: float, digest: bytes,
               pixels: bytes) -> bytes:
    """Reference-compatible packing of an existing frame (service.py:48-53)."""
    return FRAME_HEADER.pack(FRAME_MAGIC, FRAME_VERSION, sequence, width, height, render_ms,
                             digest) + pixels


def render_message(volume: Volume, camera: Camera, params: RenderParams, config: FilterConfig,
                   histogram: HistogramModel | None, sequence: int) -> memoryview:
    """One framed frame: header + W*H grey pixels, rendered on the B200."""
    t0 = time.perf_counter()
    config = _check_render_args(config, histogram, None)
    _lib.require_device()
    dev = device_volume(volume)
    rs, rp, fc = _native(camera, params, config, histogram, True)
    W, H = params.width, params.height
    hdr = FRAME_HEADER.size
    msg = _lib.pinned.array((hdr + W * H,), np.uint8)
    out = _lib.vx_render_out()
    out.pixels = msg.ctypes.data + hdr
    _lib.call("vx_render", dev.handle, C.byref(rs), C.byref(rp), C.byref(fc), None, C.byref(out))
    render_ms = (time.perf_counter() - t0) * 1000.0
    FRAME_HEADER.pack_into(msg, 0, FRAME_MAGIC, FRAME_VERSION, sequence, W, H, render_ms,
                           config.digest())
    return memoryview(msg)


def unpack_header(message) -> dict:
    magic, version, sequence, width, height, render_ms, digest = FRAME_HEADER.unpack_from(message, 0)
    return {"magic": magic, "version": version, "sequence": sequence, "width": width,
            "height": height, "render_ms": render_ms, "digest": digest}
