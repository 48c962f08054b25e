"""Per-warp timeline of one K4 frame (debug build with -DVX_WARP_TIMING):
    VOXB200_LIB=.../libvoxb200_wt.so python scripts/warp_times.py [n] [kind] [W]

The timed frame is a diagnostics frame (same schedule: tile order + split
rays), so each warp's timing, tile, segment count and march counters come
from the same launch."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import _lib, phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.render import render_detail
from paper_1807_03119_b200.volume import _attach, generate_phantom_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kind = sys.argv[2] if len(sys.argv) > 2 else "local-cluster"
W = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
spec = phantoms.insect_phantom_spec(n)
dev = generate_phantom_device(spec)
h = model_from_counts(dev.counts())
v = _attach(vx.Volume(dims=spec.dims, data=np.zeros(1, np.uint8).repeat(n ** 3)), dev)
object.__setattr__(v, "_content_hash", "x")
cam = vx.orbit_camera(v)
p = vx.RenderParams(width=W, height=W)
cfg = vx.FilterConfig(kind=vx.FilterKind.from_name(kind)).resolve_threshold(h)
for _ in range(10):  # the schedule (order from frame k-2's costs) converges over a few frames
    d = render_detail(v, cam, p, cfg, h, diagnostics=True)
nmax = 2 * W * W // 32
lib = _lib.load()
t0 = np.zeros(nmax, np.uint64); t1 = np.zeros(nmax, np.uint64); info = np.zeros(nmax, np.uint32)
lib.vx_debug_warp_times(C.c_void_p(t0.ctypes.data), C.c_void_p(t1.ctypes.data),
                        C.c_void_p(info.ctypes.data), nmax)
dg = np.zeros(nmax * 9, np.uint32)
lib.vx_debug_warp_diag(C.c_void_p(dg.ctypes.data), nmax)
dg = dg.reshape(nmax, 9)
# warps of this frame only (spare blocks of the reserve leave no record)
# records of earlier frames (slots this launch did not use) end before this
# frame's first warp: keep everything after the largest start gap
ts = np.sort(t0[t0 > 0].astype(np.float64))
cut = ts[np.argmax(np.diff(ts)) + 1] if len(ts) > 1 and np.diff(ts).max() > 20e3 else ts[0]
keep = (t0 > 0) & (t0.astype(np.float64) >= cut)
idx = np.nonzero(keep)[0]
t0, t1, info, dg = t0[keep], t1[keep], info[keep], dg[keep]
sm, nseg, part, tile = info & 0xff, (info >> 8) & 0xf, (info >> 12) & 0xf, info >> 16
base = t0.min()
s = (t0 - base).astype(np.float64) / 1e3
e = (t1 - base).astype(np.float64) / 1e3
dur = e - s
print(f"kernel span {e.max():.1f} us; warps {len(dur)}; dur p50 {np.median(dur):.2f} p90 "
      f"{np.percentile(dur, 90):.2f} p99 {np.percentile(dur, 99):.2f} max {dur.max():.2f} us; "
      f"sum {dur.sum() / 1e3:.1f} ms-warp")
print(f"ideal (sum / (148*32 slots)) {dur.sum() / (148 * 32):.1f} us; last warp start {s.max():.1f} us")
for k in (8, 4, 2, 1):
    m = nseg == k
    if m.any():
        print(f"  nseg {k}: {m.sum()} warps ({len(np.unique(tile[m]))} tiles), dur max {dur[m].max():.1f} "
              f"p50 {np.median(dur[m]):.1f} us, start max {s[m].max():.1f} us")
end = np.array([e[sm == k].max() for k in np.unique(sm)])
print(f"per-SM last end: min {end.min():.1f} median {np.median(end):.1f} max {end.max():.1f} us")
names = ("lookups", "inchunk", "chunks", "unused", "groups", "filters", "hits", "iters", "max_iters")
top = np.argsort(-dur)[:8]
tiles_x = W // 8
for w in top:
    ty, tx = divmod(int(tile[w]), tiles_x)
    print(f"  warp {idx[w]}: dur {dur[w]:.1f} us start {s[w]:.1f} tile ({ty * 16},{tx * 8}) nseg {nseg[w]} "
          f"part {part[w]} sm {sm[w]} | " + " ".join(f"{k}={int(x)}" for k, x in zip(names, dg[w])))
med = np.median(dg, axis=0)
print("  median warp: " + " ".join(f"{k}={x:.0f}" for k, x in zip(names, med)))
# occupancy over time: resident warps per 5% of the span
edges = np.linspace(0, e.max(), 21)
occ = [int(((s < b) & (e > a)).sum()) for a, b in zip(edges[:-1], edges[1:])]
print("warps alive per 5% of the span:", occ)
