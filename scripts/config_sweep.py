"""Time every BASELINE.json config on one B200 (device-resident, CUDA events,
L2 flushed between reps) and print one JSON object.

    python scripts/config_sweep.py [--reps 20] > profiles/r1_config_sweep.json

C1 spot_64 @256^2 (six filters), C2/C3 insect_512 @1024^2 (six filters +
entropy), C4 insect_2048 @2048^2 (local cluster), C5 K1+K2 over 256^3..4096^3.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())

import numpy as np
import torch

import paper_1807_03119_b200 as vx
from paper_1807_03119_b200 import _lib, phantoms
from paper_1807_03119_b200.filters import native_config
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.metrics import entropy_from_counts
from paper_1807_03119_b200.render import native_params, ray_setup
from paper_1807_03119_b200.volume import _attach, generate_phantom_device

KINDS = ("none", "mean", "sigma", "entropy", "okada", "local-cluster")


def timed(fn, reps, flush):
    stream = torch.cuda.current_stream()
    out = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            out.append(a.elapsed_time(b))
    return statistics.median(out)


def frame_runner(dvol, hist, W, kind, stream):
    v = _attach(vx.Volume(dims=dvol.dims, data=np.zeros(1, np.uint8).repeat(int(np.prod(dvol.dims)))),
                dvol) if False else None
    cam = vx.orbit_camera(type("V", (), {"dims": dvol.dims})())
    params = vx.RenderParams(width=W, height=W)
    kw = {"entropy_threshold": 0.5} if kind == "entropy" else {}
    cfg = vx.FilterConfig(kind=vx.FilterKind.from_name(kind), **kw).resolve_threshold(hist)
    rs, rp, fc = ray_setup(cam, W, W), native_params(params), native_config(cfg, hist)
    pixels = torch.zeros(W * W, dtype=torch.uint8, device="cuda")
    small = torch.zeros(260, dtype=torch.int64, device="cuda")
    out = _lib.vx_render_out()
    out.pixels = pixels.data_ptr()
    out.image_hist = small.data_ptr()
    out.hit_count = small.data_ptr() + 256 * 8
    out.samples = small.data_ptr() + 257 * 8
    out.trunc_flag = small.data_ptr() + 258 * 8
    sp = C.c_void_p(stream.cuda_stream)

    def run():
        small.zero_()
        _lib.call("vx_render_device", dvol.handle, C.byref(rs), C.byref(rp), C.byref(fc), None,
                  C.byref(out), sp)

    return run, small


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--skip-4096", action="store_true")
    ap.add_argument("--frames-only", action="store_true", help="skip the C5 histogram sweep")
    ap.add_argument("--hist-only", action="store_true", help="only the C5 histogram sweep")
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {"device": torch.cuda.get_device_name(0), "reps": args.reps}

    def frames(name, spec, W, kinds):
        dvol = generate_phantom_device(spec)
        hist = model_from_counts(dvol.counts())
        rows = {}
        for kind in kinds:
            run, small = frame_runner(dvol, hist, W, kind, stream)
            ms = timed(run, args.reps, flush)
            sm = small.cpu().numpy()
            rows[kind] = {"ms": ms, "fps": 1000.0 / ms, "hits": int(sm[256]),
                          "samples": int(sm[257]),
                          "entropy_bits": entropy_from_counts(sm[:256], W * W)}
        res[name] = {"volume": list(spec.dims), "image": [W, W], "otsu_T": hist.otsu_threshold,
                     "filters": rows}
        dvol.free()

    if not args.hist_only:
        frames("C1_spot64_256", phantoms.spot_phantom_spec(64), 256, KINDS)
        frames("C2_C3_insect512_1024", phantoms.insect_phantom_spec(512), 1024, KINDS)
        frames("bench_insect1024_1024", phantoms.insect_phantom_spec(1024), 1024,
               ("local-cluster",))
        frames("C4_insect2048_2048", phantoms.insect_phantom_spec(2048), 2048, ("local-cluster",))

    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists(
        "MEASURED_PEAKS.json") else 6650.0
    sweep = {}
    for edge in (() if args.frames_only else (256, 512, 1024, 2048, 4096)):
        n = edge ** 3
        if edge == 4096 and (args.skip_4096 or torch.cuda.mem_get_info()[0] < n + (2 << 30)):
            continue
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        # bimodal CT-like bytes (device generator)
        spec = vx.PhantomSpec(dims=(edge, edge, edge),
                              shapes=(vx.Shape(kind="sphere", center=((edge - 1) / 2,) * 3,
                                               radius=edge * 0.3125, intensity=200),),
                              noise_sigma=10.0, rng_seed=5)
        from paper_1807_03119_b200.volume import _phantom_args

        table, ns, seed, spots, k = _phantom_args(spec)
        _lib.call("vx_phantom_device", C.c_void_p(t.data_ptr()), edge, edge, edge,
                  _lib.ptr(table), ns, 10.0, seed, _lib.ptr(spots), k, 255,
                  C.c_void_p(stream.cuda_stream))
        counts = torch.zeros(256, dtype=torch.int64, device="cuda")
        dT = torch.zeros(1, dtype=torch.int32, device="cuda")
        sp = C.c_void_p(stream.cuda_stream)

        def run():
            _lib.call("vx_histogram_otsu_device", C.c_void_p(t.data_ptr()), n,
                      C.c_void_p(counts.data_ptr()), C.c_void_p(dT.data_ptr()), sp)

        ms = timed(run, args.reps, flush)
        gbs = n / (ms * 1e-3) / 1e9
        sweep[f"{edge}^3"] = {"bytes": n, "ms": ms, "GB/s": gbs, "frac_of_hbm": gbs / peak,
                              "otsu_T": int(dT.item())}
        del t
    res["C5_hist_sweep"] = sweep
    res["hbm_peak_gbs"] = peak
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
