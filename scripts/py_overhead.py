"""Host-side cost of render_frame per call (cProfile over warm bench frames):
where the Python microseconds around the C call go."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.volume import _attach, generate_phantom_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
spec = phantoms.insect_phantom_spec(n)
dev = generate_phantom_device(spec)
h = model_from_counts(dev.counts())
v = _attach(vx.Volume(dims=spec.dims, data=np.zeros(1, np.uint8).repeat(n ** 3)), dev)
object.__setattr__(v, "_content_hash", "x")
cam = vx.orbit_camera(v)
p = vx.RenderParams(width=1024, height=1024)
cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER).resolve_threshold(h)
for _ in range(20):
    vx.render_frame(v, cam, p, cfg, h)
N = 2000
t0 = time.perf_counter()
for _ in range(N):
    vx.render_frame(v, cam, p, cfg, h)
wall = (time.perf_counter() - t0) / N * 1e6
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    vx.render_frame(v, cam, p, cfg, h)
pr.disable()
print(f"render_frame wall {wall:.1f} us/frame")
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
