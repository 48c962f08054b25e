import json
import os
import sys
import traceback

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_1807_03119_b200 as vx
from oracle.rng_np import generate_phantom_np
from paper_1807_03119_b200.render import render_detail
from pathlib import Path
GOLDEN = Path('tests/golden')
def golden(n):
    return np.load(GOLDEN / n)

step = sys.argv[1] if len(sys.argv) > 1 else "all"

if step in ("filt", "all"):
    try:
        from paper_1807_03119_b200.filters import apply_filter, apply_filter_batch
        g = golden("filters.npz")
        vol, pts = g["volumes"][0], g["coords"][0]
        v = vx.Volume(dims=(9, 9, 9), data=vol)
        h = vx.build_histogram(v)
        cfg = vx.FilterConfig(kind=vx.FilterKind.NONE)
        print("batch", apply_filter_batch(v, pts[:, 0], pts[:, 1], pts[:, 2], cfg, h), flush=True)
        print("scalar", apply_filter(v, *map(int, pts[0]), cfg, h), flush=True)
    except Exception:
        traceback.print_exc()

if step in ("speckle", "all"):
    meta = json.loads((GOLDEN / "phantoms.json").read_text())
    g = golden("frames_small.npz")
    for name in ("speckle_128", "spot_64"):
        spec = vx.PhantomSpec.from_json(meta[name]["spec"])
        host = generate_phantom_np(meta[name]["spec"])
        for src in ("host", "device"):
            if src == "host":
                v = vx.Volume(dims=spec.dims, data=host)
            else:
                v = vx.generate_phantom(spec)
                print(name, "device phantom equal:", np.array_equal(v.data, host),
                      int((v.data != host).sum()), flush=True)
            h = vx.build_histogram(v)
            cam = vx.orbit_camera(v)
            size = g[f"{name}__none__pixels"].shape[0]
            p = vx.RenderParams(width=size, height=size)
            for kind in ("none", "local-cluster"):
                for skip in (True, False):
                    d = render_detail(v, cam, p, vx.FilterConfig(kind=vx.FilterKind.from_name(kind)), h,
                                      diagnostics=True, skip=skip)
                    want = g[f"{name}__{kind}__voxel"].astype(np.int32)
                    bad = np.any(d.hit_voxel != want, axis=1)
                    print(name, src, kind, "skip", skip, "voxel mismatches", int(bad.sum()),
                          "pixel mism", int((d.pixels != g[f"{name}__{kind}__pixels"]).sum()),
                          "T", h.otsu_threshold, "samples", d.samples, flush=True)
                    if bad.any():
                        idx = np.nonzero(bad)[0][:5]
                        for i in idx:
                            print("   px", i, "got", d.hit_voxel[i], "want", want[i], flush=True)
