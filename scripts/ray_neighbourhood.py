"""Accepted voxels (raw >= thr and LC >= T) near a slow bench ray."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.render import primary_ray_dirs, ray_box_spans
from paper_1807_03119_b200.volume import _attach, generate_phantom_device

n = 1024
spec = phantoms.insect_phantom_spec(n)
dev = generate_phantom_device(spec)
host = dev.read()
h = model_from_counts(dev.counts())
v = _attach(vx.Volume(dims=spec.dims, data=host), dev)
object.__setattr__(v, "_content_hash", "x")
cam = vx.orbit_camera(v)
cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER).resolve_threshold(h)
thr = int(np.ceil(cfg.threshold))
dirs = primary_ray_dirs(cam, 1024, 1024)
te, tx = ray_box_spans(np.asarray(cam.position), dirs, spec.dims)
print("shapes:", [(s.kind, s.center, s.radius, s.extent, s.intensity) for s in spec.shapes[:12]], len(spec.shapes))
for (r, c) in [(624, 480), (384, 432)]:
    i = r * 1024 + c
    o = np.asarray(cam.position) + 0.5
    ts = np.arange(te[i], tx[i], 2.0)
    P = o + ts[:, None] * dirs[i]
    R = 24
    pts = set()
    for p in P[::4]:
        lo = np.maximum(np.floor(p).astype(int) - R, 0)
        hi = np.minimum(np.floor(p).astype(int) + R, n - 1)
        sub = host[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
        zz, yy, xx = np.nonzero(sub >= thr)
        for a, b, cc in zip(xx + lo[0], yy + lo[1], zz + lo[2]):
            pts.add((int(a), int(b), int(cc)))
    pts = np.array(sorted(pts), dtype=np.int64).reshape(-1, 3)
    print(f"ray ({r},{c}): {len(pts)} candidates within {R} of the path")
    if len(pts):
        from paper_1807_03119_b200.filters import apply_filter_batch
        f = apply_filter_batch(v, pts[:, 0], pts[:, 1], pts[:, 2], cfg, h)
        acc = pts[f >= cfg.threshold]
        # distance from the ray
        def dist(q):
            w = q + 0.5 - o
            tt = w @ dirs[i]
            return np.linalg.norm(w - tt[:, None] * dirs[i], axis=1), tt
        dd, tt = dist(acc.astype(float))
        print(f"  accepted {len(acc)}; raw values {np.bincount(host[acc[:,2],acc[:,1],acc[:,0]] // 32, minlength=8)} (by 32s)")
        order = np.argsort(tt)
        for q in order[:: max(1, len(order) // 15)]:
            print(f"   voxel {tuple(acc[q])} raw {host[acc[q][2], acc[q][1], acc[q][0]]} dist {dd[q]:.1f} t {tt[q]:.0f}")
