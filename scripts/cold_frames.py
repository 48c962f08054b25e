"""Cold-frame wall times on the bench volume: frame 1 of a volume (candidate
distance map of thr), frame 2 (the filter's accepted-cell map), frame 3+
(warm), and a second filter setting's first two frames."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.volume import _attach, generate_phantom_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
t0 = time.perf_counter()
spec = phantoms.insect_phantom_spec(n)
dev = generate_phantom_device(spec)
torch.cuda.synchronize()
t1 = time.perf_counter()
h = model_from_counts(dev.counts())
v = _attach(vx.Volume(dims=spec.dims, data=np.zeros(1, np.uint8).repeat(n ** 3)), dev)
object.__setattr__(v, "_content_hash", "x")
cam = vx.orbit_camera(v)
p = vx.RenderParams(width=1024, height=1024)
print(f"volume {n}^3 generated + replica + K1 in {(t1 - t0) * 1e3:.1f} ms")
for kind in ("local-cluster", "mean", "local-cluster"):
    cfg = vx.FilterConfig(kind=vx.FilterKind.from_name(kind)).resolve_threshold(h)
    ts = []
    for i in range(4):
        torch.cuda.synchronize()
        a = time.perf_counter()
        vx.render_frame(v, cam, p, cfg, h)
        ts.append((time.perf_counter() - a) * 1e3)
    print(kind, " ".join(f"{x:.2f}" for x in ts), "ms")
