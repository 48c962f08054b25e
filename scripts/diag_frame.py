"""Per-frame march statistics of the bench workload (diagnostics build path)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.render import render_detail
from paper_1807_03119_b200.volume import generate_phantom_device, _attach

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kind = sys.argv[2] if len(sys.argv) > 2 else "local-cluster"
spec = phantoms.insect_phantom_spec(n)
dev = generate_phantom_device(spec)
h = model_from_counts(dev.counts())
v = _attach(vx.Volume(dims=spec.dims, data=np.zeros(1, np.uint8).repeat(n**3)), dev)
cam = vx.orbit_camera(v)
p = vx.RenderParams(width=1024, height=1024)
cfg = vx.FilterConfig(kind=vx.FilterKind.from_name(kind), **({"entropy_threshold": 0.5} if kind == "entropy" else {}))
for rep in range(3):  # raw map, accepted-cell map (built), accepted-cell map (cached)
    t0 = time.perf_counter(); d = render_detail(v, cam, p, cfg, h, diagnostics=True); dt = time.perf_counter() - t0
    print(kind, n, "rep", rep, "samples", d.samples, "hits", d.hit_count, d.diag, f"{dt*1e3:.2f} ms wall", flush=True)
