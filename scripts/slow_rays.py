"""Inspect the rays of a slow K4 warp (bench frame): spans, hits, and the
accepted-cell distance along each ray."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.render import render_detail, primary_ray_dirs, ray_box_spans
from paper_1807_03119_b200.volume import _attach, generate_phantom_device

n = 1024
spec = phantoms.insect_phantom_spec(n)
dev = generate_phantom_device(spec)
host = dev.read()
h = model_from_counts(dev.counts())
v = _attach(vx.Volume(dims=spec.dims, data=host), dev)
object.__setattr__(v, "_content_hash", "x")
cam = vx.orbit_camera(v)
p = vx.RenderParams(width=1024, height=1024)
cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER).resolve_threshold(h)
d = render_detail(v, cam, p, cfg, h, diagnostics=True)
dirs = primary_ray_dirs(cam, 1024, 1024)
te, tx = ray_box_spans(np.asarray(cam.position), dirs, spec.dims)
T = cfg.threshold
thr = int(np.ceil(T))
o = np.asarray(cam.position) + 0.5
for (r0, c0) in [(624, 480), (412, 568), (540, 360), (384, 432)]:
    print(f"--- warp rows {r0}..{r0+3} cols {c0}..{c0+7}")
    for r in range(r0, r0 + 4):
        for c in (c0, c0 + 3, c0 + 7):
            i = r * 1024 + c
            hv = d.hit_voxel[i]
            # walk the ray in float64 (approximate) and count candidate samples before the hit
            tend = d.hit_t[i] if hv[0] >= 0 else tx[i]
            ts = np.arange(te[i], tend, 0.5)
            pos = np.trunc(o + ts[:, None] * dirs[i]).astype(np.int64)
            ok = ((pos >= 0) & (pos < n)).all(1)
            vals = np.zeros(len(ts), np.int64)
            q = pos[ok]
            vals[ok] = host[q[:, 2], q[:, 1], q[:, 0]]
            cand = int((vals >= thr).sum())
            print(f"  px ({r},{c}) hit {tuple(hv)} t {d.hit_t[i]:.1f} span [{te[i]:.1f},{tx[i]:.1f}] "
                  f"samples {len(ts)} candidates {cand}")
