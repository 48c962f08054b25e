"""Where the end-to-end frame time goes (bench frame): render_frame vs the
bare C-ABI call vs the device-only launch, per-frame wall clock."""
import ctypes as C, os, statistics, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import _lib, phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.render import _native
from paper_1807_03119_b200.volume import _attach, generate_phantom_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
spec = phantoms.insect_phantom_spec(n)
dev = generate_phantom_device(spec)
h = model_from_counts(dev.counts())
v = _attach(vx.Volume(dims=spec.dims, data=np.zeros(1, np.uint8).repeat(n ** 3)), dev)
object.__setattr__(v, "_content_hash", "x")
cam = vx.orbit_camera(v)
p = vx.RenderParams(width=1024, height=1024)
cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER).resolve_threshold(h)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def per_frame(fn, reps=50, do_flush=True, dist=False):
    out = []
    for i in range(reps + 5):
        if do_flush:
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        if i >= 5:
            out.append((t1 - t0) * 1e3)
    if dist:
        q = sorted(out)
        return (f"median {statistics.median(q):.4f} mean {statistics.mean(q):.4f} "
                f"p10 {q[len(q) // 10]:.4f} p90 {q[9 * len(q) // 10]:.4f} max {q[-1]:.4f}")
    return statistics.median(out)


rs, rp, fc = _native(cam, p, cfg, h, True)
pix = _lib.pinned.array((1024, 1024), np.uint8)
out = _lib.vx_render_out()
out.pixels = pix.ctypes.data


def bare():
    _lib.call("vx_render", dev.handle, C.byref(rs), C.byref(rp), C.byref(fc), None, C.byref(out))


dpix = torch.empty(1024 * 1024, dtype=torch.uint8, device="cuda")
small = torch.zeros(260, dtype=torch.int64, device="cuda")
dout = _lib.vx_render_out()
dout.pixels = dpix.data_ptr()
dout.image_hist = small.data_ptr()
dout.hit_count = small.data_ptr() + 2048
dout.trunc_flag = small.data_ptr() + 258 * 8
stream = torch.cuda.current_stream()


def devonly():
    small.zero_()
    _lib.call("vx_render_device", dev.handle, C.byref(rs), C.byref(rp), C.byref(fc), None,
              C.byref(dout), C.c_void_p(stream.cuda_stream))
    torch.cuda.synchronize()


for name, fn in [("render_frame", lambda: vx.render_frame(v, cam, p, cfg, h)), ("bare vx_render", bare),
                 ("device launch+sync", devonly)]:
    print(f"{name:22s} flushed {per_frame(fn):.4f} ms   warm {per_frame(fn, do_flush=False):.4f} ms")

for name, fn in [("render_frame", lambda: vx.render_frame(v, cam, p, cfg, h)), ("bare vx_render", bare),
                 ("device launch+sync", devonly)]:
    print(f"{name:22s} flushed x200: {per_frame(fn, reps=200, dist=True)}")
