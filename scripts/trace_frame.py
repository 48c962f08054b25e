"""Host phases of vx_render (VOXB200_TRACE=1) for a few warm bench frames."""
import os, sys
os.environ["VOXB200_TRACE"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.volume import _attach, generate_phantom_device

spec = phantoms.insect_phantom_spec(1024)
dev = generate_phantom_device(spec)
h = model_from_counts(dev.counts())
v = _attach(vx.Volume(dims=spec.dims, data=np.zeros(1, np.uint8).repeat(1024 ** 3)), dev)
object.__setattr__(v, "_content_hash", "x")
cam = vx.orbit_camera(v)
p = vx.RenderParams(width=1024, height=1024)
cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER).resolve_threshold(h)
for i in range(8):
    sys.stderr.write(f"--- frame {i}\n")
    vx.render_frame(v, cam, p, cfg, h)
