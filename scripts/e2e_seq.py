import os, sys, time, gc
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import _lib, phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.volume import _attach, generate_phantom_device
spec = phantoms.insect_phantom_spec(1024)
dvol = generate_phantom_device(spec)
hist = model_from_counts(dvol.counts())
host = dvol.read()
volume = _attach(vx.Volume(dims=spec.dims, data=host), dvol)
volume.content_hash()
cam = vx.orbit_camera(volume)
params = vx.RenderParams(width=1024, height=1024)
cfg = vx.FilterConfig(kind=vx.FilterKind.LOCAL_CLUSTER).resolve_threshold(hist)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rnd in range(3):
    for _ in range(3):
        vx.render_frame(volume, cam, params, cfg, hist)
    ts, dev, nl = [], [], []
    from paper_1807_03119_b200.render import frame_timing
    with frame_timing():
        for _ in range(20):
            flush.zero_(); torch.cuda.synchronize()
            _lib.launches(reset=True)
            t0 = time.perf_counter(); f = vx.render_frame(volume, cam, params, cfg, hist); ts.append((time.perf_counter() - t0) * 1e3)
            dev.append(f.timing["device_ms"]); nl.append(_lib.launches())
    print(rnd, "wall", " ".join(f"{t:.3f}" for t in ts))
    print(rnd, "dev ", " ".join(f"{t:.3f}" for t in dev))
    print(rnd, "launches", nl)
