"""Where does an orbiting frame's time go?  Host struct building vs device
K4 time vs wall, for a static camera and for 1 degree/frame azimuth steps."""
import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.render import ray_setup, frame_timing
from paper_1807_03119_b200.volume import _attach, generate_phantom_device

spec = phantoms.insect_phantom_spec(1024)
dv = generate_phantom_device(spec)
h = model_from_counts(dv.counts())
v = _attach(vx.Volume(dims=spec.dims, data=dv.read()), dv)
v.content_hash()
p = vx.RenderParams(width=1024, height=1024)
cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cams = [vx.orbit_camera(v, azimuth_deg=45.0 + k) for k in range(100)]
t0 = time.perf_counter()
for c in cams:
    ray_setup(c, 1024, 1024)
print(f"ray_setup host: {(time.perf_counter() - t0) / len(cams) * 1e6:.1f} us/frame")
for _ in range(5):
    vx.render_frame(v, cams[0], p, cfg, h)
def run(cs, label):
    wall, dev = [], []
    with frame_timing():
        for c in cs:
            flush.zero_(); torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = vx.render_frame(v, c, p, cfg, h)
            wall.append((time.perf_counter() - t0) * 1e3); dev.append(f.timing["device_ms"])
    print(f"{label}: wall p50 {statistics.median(wall):.3f} ms, device p50 {statistics.median(dev):.3f} "
          f"max {max(dev):.3f} ms")
    return dev
run([cams[0]] * 100, "static")
d1 = run(cams, "orbit 1deg")
run(cams, "orbit again (same cameras, warm orders)")
# per-azimuth static device time: is the orbit path just costlier views?
stat = []
for c in cams[::10]:
    with frame_timing():
        for _ in range(4):
            f = vx.render_frame(v, c, p, cfg, h)
    stat.append(f.timing["device_ms"])
print("static device ms at az 45,55,..:", " ".join(f"{x:.3f}" for x in stat))
print("orbit  device ms at az 45,55,..:", " ".join(f"{x:.3f}" for x in d1[::10]))
# each orbit camera rendered three times, the third timed: a repeated camera
# renders in the order of frame k-2, the same camera's first render (zero
# staleness)
dev2 = []
with frame_timing():
    for c in cams:
        vx.render_frame(v, c, p, cfg, h)
        vx.render_frame(v, c, p, cfg, h)
        flush.zero_(); torch.cuda.synchronize()
        f = vx.render_frame(v, c, p, cfg, h)
        dev2.append(f.timing["device_ms"])
print(f"orbit, each camera three times (3rd timed): device p50 {statistics.median(dev2):.3f} max {max(dev2):.3f} ms")
