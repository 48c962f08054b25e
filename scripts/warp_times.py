"""Per-warp timeline of one K4 frame (debug build with -DVX_WARP_TIMING):
    VOXB200_LIB=.../libvoxb200_wt.so python scripts/warp_times.py [n] [kind]"""
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
for _ in range(3):
    d = render_detail(v, cam, p, cfg, h)
nw = W * W // 32
lib = _lib.load()
t0 = np.zeros(nw, np.uint64); t1 = np.zeros(nw, np.uint64); sm = np.zeros(nw, np.uint32)
lib.vx_debug_warp_times(C.c_void_p(t0.ctypes.data), C.c_void_p(t1.ctypes.data),
                        C.c_void_p(sm.ctypes.data), nw)
base = t0.min()
s = (t0 - base).astype(np.float64) / 1e3
e = (t1 - base).astype(np.float64) / 1e3
dur = e - s
print(f"kernel span {e.max():.1f} us; warps {nw}; dur p50 {np.median(dur):.2f} p90 {np.percentile(dur,90):.2f} "
      f"p99 {np.percentile(dur,99):.2f} max {dur.max():.2f} us; sum {dur.sum()/1e3:.1f} ms-warp")
print(f"ideal (sum / (148*32 slots)) {dur.sum()/(148*32):.1f} us; last warp start {s.max():.1f} us")
busy = np.zeros(sm.max() + 1)
end = np.zeros(sm.max() + 1)
for k in range(len(busy)):
    m = sm == k
    end[k] = e[m].max() if m.any() else 0
print(f"per-SM last end: min {end.min():.1f} median {np.median(end):.1f} max {end.max():.1f} us")
# warp index -> tile position: block b = w // 4 covers tile b (8x16), warp w%4 the rows 4*(w%4)..
tiles_x = W // 8
b = np.arange(nw) // 4
ty, tx = b // tiles_x, b % tiles_x
row = ty * 16 + (np.arange(nw) % 4) * 4
col = tx * 8
top = np.argsort(-dur)[:6]
for w in top:
    print(f"  warp {w}: dur {dur[w]:.1f} us start {s[w]:.1f} rows {row[w]}..{row[w]+3} cols {col[w]}..{col[w]+7} sm {sm[w]}")
# duration by image band (64 rows)
img = np.zeros((W // 4, W // 8))
img[row // 4, col // 8] = dur
bands = img.reshape(W // 64, 16, W // 8).sum(axis=(1, 2)) / 1e3
print("ms-warp per 64-row band:", " ".join(f"{x:.1f}" for x in bands))
np.save("gpurun_out/warp_dur.npy", img)
# per-warp march statistics (diagnostics frame; the warp deal is identical)
d = render_detail(v, cam, p, cfg, h, diagnostics=True)
dg = np.zeros(nw * 9, np.uint32)
lib.vx_debug_warp_diag(C.c_void_p(dg.ctypes.data), nw)
dg = dg.reshape(nw, 9)
names = ("lookups", "inchunk", "chunks", "unused", "groups", "filters", "hits", "iters", "max_iters")
print("slowest warps (timing frame) statistics (diag frame):")
for w in top[:8]:
    print(f"  warp {w}: " + " ".join(f"{k}={int(x)}" for k, x in zip(names, dg[w])))
med = np.median(dg, axis=0)
print("  median warp: " + " ".join(f"{k}={x:.0f}" for k, x in zip(names, med)))
