#!/usr/bin/env python
"""Headline benchmark: filtered frames/s at 1024^2 on a 1024^3 CT volume (B200),
plus the Otsu histogram throughput against HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (sort-first, tiles split)

Workload (BASELINE.json metric): the CT-like insect phantom
(C2 recipe scaled to 1024^3, generated on the device by K7), Otsu threshold
from the device histogram (K1 + K2), orbit camera defaults, 1024x1024 image,
local-cluster filter (M=3, d=1), Sobel + Phong.  A step is one full frame.

value      frames/s with the volume resident in HBM; per-step CUDA events on
           the launch stream around the frame (render kernel [+ NCCL reduce
           for N>1]); L2 flushed (256 MiB write) between steps, outside the
           events; max over ranks.
e2e        the same frames through the public drop-in API
           (paper_1807_03119_b200.render_frame) with host outputs: camera /
           params uploaded and the 1 MiB frame + histogram read back each step.
roofline   dominant kernel (K4 raycast): SURVEY §8d algorithmic bytes
           (N voxels + W*H) / kernel time vs MEASURED_PEAKS hbm_gbs.
cpu_baseline  oracle/ C restatement of the reference (1 thread) on a bounded
           row sample of the same frame, extrapolated to frames/s.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "filtered frames/s (ms/frame) at 1024² on 1024³ CT; Otsu hist GB/s vs HBM"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=1024, help="volume edge (voxels)")
    ap.add_argument("--image", type=int, default=1024, help="image edge (pixels)")
    ap.add_argument("--filter", default="local-cluster")
    ap.add_argument("--no-skip", action="store_true", help="disable exact empty-space skipping")
    ap.add_argument("--cpu-rows", type=int, default=16, help="CPU baseline: every k-th row")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) polled every 2 ms from a thread; falls back to
    `nvidia-smi -lms 10` if NVML is unavailable.
    """

    REASONS = {"hw_slowdown": "nvmlClocksThrottleReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksThrottleReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksThrottleReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksThrottleReasonSwPowerCap"}

    def __init__(self, device: int):
        self.device = device
        self.sm: list[float] = []
        self.max_mhz = None
        self.reasons: set[str] = set()
        self._stop = threading.Event()
        self._thread = None
        self._proc = None

    def _nvml_loop(self, nv, h, masks):
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                for name, m in masks.items():
                    if r & m:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            idx = self.device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis and vis.split(",")[0].strip().isdigit():
                idx = int(vis.split(",")[self.device])
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            masks = {k: getattr(nv, v) for k, v in self.REASONS.items()}
            self._thread = threading.Thread(target=self._nvml_loop, args=(nv, h, masks), daemon=True)
            self._thread.start()
            while not self.sm and self._thread.is_alive():
                time.sleep(0.001)
        except Exception:
            self._start_smi()
        return self

    def _start_smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={fields}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def read():
                names = list(self.REASONS)
                for line in self._proc.stdout:
                    parts = [p.strip() for p in line.split(",")]
                    try:
                        self.sm.append(float(parts[0]))
                        self.max_mhz = float(parts[1])
                    except (ValueError, IndexError):
                        continue
                    for n, v in zip(names, parts[2:6]):
                        if v.lower() == "active":
                            self.reasons.add(n)

            self._thread = threading.Thread(target=read, daemon=True)
            self._thread.start()
            t0 = time.time()
            while not self.sm and time.time() - t0 < 5:
                time.sleep(0.005)
        except Exception:
            self._proc = None

    def __exit__(self, *exc):
        self._stop.set()
        if self._proc:
            self._proc.terminate()
        if self._thread:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def cpu_baseline(volume_host: np.ndarray, cam_vec, W, H, kind, T, hist, row_step, threads):
    from oracle import oracle as orc

    orc.build()
    t0 = time.perf_counter()
    r = orc.render(volume_host, cam_vec, W, H, kind=kind, threshold=T,
                   sigma_band=2.0 * hist.global_sigma, probabilities=hist.probabilities,
                   row_step=row_step, threads=threads, diagnostics=False)
    dt = time.perf_counter() - t0
    rows = len(range(0, H, row_step))
    frac = rows / H
    return {"value": frac / dt, "unit": "frames/s", "cores": threads, "kind": "port",
            "sample": f"oracle/vxoracle.c render of every {row_step}th row ({rows}/{H} rows) of the "
                      f"same frame, {dt:.2f}s, extrapolated to a full frame",
            "seconds": dt, "samples_taken": r["samples"]}


# ------------------------------------------------------------------------------------


def run_reference(args):
    """--impl reference: the oracle C restatement of the reference CPU path."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc
    from paper_1807_03119_b200 import phantoms

    orc.build()
    threads = orc.max_threads()
    spec = phantoms.insect_phantom_spec(args.size).to_json()
    t0 = time.perf_counter()
    vol = orc.phantom(spec, threads=threads)
    gen_s = time.perf_counter() - t0
    counts = orc.hist256(vol)
    hm = orc.histogram_model(counts)
    pos, look = orc.orbit(vol.shape[::-1])
    W = H = args.image
    cam = orc.cam_vector(pos, look, W, H)
    row_step = max(1, args.cpu_rows)
    rows = len(range(0, H, row_step))
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        orc.render(vol, cam, W, H, kind=args.filter, threshold=float(hm["otsu"]),
                   sigma_band=2.0 * hm["global_sigma"], probabilities=hm["probabilities"],
                   row_step=row_step, threads=threads, diagnostics=False)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    per_frame = statistics.mean(times) * H / rows
    value = 1.0 / per_frame
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_frame * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"insect_{args.size}^3 @ {W}x{H}, {args.filter}, Otsu T",
                   "volume": [args.size] * 3, "image": [W, H], "filter": args.filter,
                   "otsu_T": hm["otsu"]},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": f"every {row_step}th row ({rows}/{H}) per step, extrapolated; "
                                   f"phantom generated on host in {gen_s:.1f}s"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1807_03119_b200 as vx
    from paper_1807_03119_b200 import _lib, phantoms
    from paper_1807_03119_b200.filters import native_config
    from paper_1807_03119_b200.histogram import model_from_counts
    from paper_1807_03119_b200.render import native_params, ray_setup
    from paper_1807_03119_b200.volume import _attach, generate_phantom_device

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    _lib.call("vx_set_device", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev_index = local

    # ---- workload (sort-first: every rank holds the full volume) ----
    spec = phantoms.insect_phantom_spec(args.size)
    t0 = time.perf_counter()
    dvol = generate_phantom_device(spec)
    gen_s = time.perf_counter() - t0
    counts = dvol.counts()
    hist = model_from_counts(counts)  # K1 (at creation) + K2
    W = H = args.image
    nvox = args.size ** 3

    # a host Volume view for the e2e / CPU legs (compact copy, read once)
    host = dvol.read()
    volume = _attach(vx.Volume(dims=spec.dims, data=host), dvol)
    volume.content_hash()
    cam = vx.orbit_camera(volume)
    params = vx.RenderParams(width=W, height=H)
    cfg = vx.FilterConfig(kind=vx.FilterKind.from_name(args.filter)).resolve_threshold(hist)
    rs = ray_setup(cam, W, H)
    rp = native_params(params, skip=not args.no_skip)
    fc = native_config(cfg, hist)
    part = _lib.vx_partition(rank, world)

    # a dedicated (non-null) stream: the C-ABI treats stream 0 as "the calling
    # thread's own stream", so torch work, events and our kernels share this one
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = C.c_void_p(stream.cuda_stream)
    pixels = torch.zeros(H * W, dtype=torch.uint8, device="cuda")
    small = torch.zeros(260, dtype=torch.int64, device="cuda")
    out = _lib.vx_render_out()
    out.pixels = pixels.data_ptr()
    out.image_hist = small.data_ptr()
    out.hit_count = small.data_ptr() + 256 * 8
    out.samples = small.data_ptr() + 257 * 8
    out.trunc_flag = small.data_ptr() + 258 * 8
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def frame():
        small.zero_()
        if world > 1:
            pixels.zero_()
        _lib.call("vx_render_device", dvol.handle, C.byref(rs), C.byref(rp), C.byref(fc),
                  C.byref(part), C.byref(out), sptr)
        if world > 1:
            dist.reduce(pixels, dst=0, op=dist.ReduceOp.SUM)
            dist.all_reduce(small[:258], op=dist.ReduceOp.SUM)

    # cold frames (wall clock, synchronised): the first builds the candidate
    # distance map of thr, the second the filter's accepted-cell map
    # (vx_render.cu get_accept_map); later frames reuse both
    cold_ms = []
    for w in range(args.warmup):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        frame()
        torch.cuda.synchronize()
        if w < 2:
            cold_ms.append((time.perf_counter() - t0) * 1000.0)
        flush.zero_()
    torch.cuda.synchronize()

    # ---- timed region: K frames, per-step events, L2 flushed between ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    kern = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    _lib.launches(reset=True)
    with ClockSampler(dev_index) as clocks:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            small.zero_()
            if world > 1:
                pixels.zero_()
            kern[i][0].record(stream)
            _lib.call("vx_render_device", dvol.handle, C.byref(rs), C.byref(rp), C.byref(fc),
                      C.byref(part), C.byref(out), sptr)
            kern[i][1].record(stream)
            if world > 1:
                dist.reduce(pixels, dst=0, op=dist.ReduceOp.SUM)
                dist.all_reduce(small[:258], op=dist.ReduceOp.SUM)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    launches = _lib.launches()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    kern_ms = [a.elapsed_time(b) for a, b in kern]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = 1000.0 / ms_per_step
    sm = small.cpu().numpy()
    trunc_flag = int(sm[258])
    samples = int(sm[257])
    hit_count = int(sm[256])

    # ---- Otsu histogram K1 over the compact 1 GiB volume (second half of the metric) ----
    hist_line = None
    if rank == 0:
        compact = torch.empty(nvox, dtype=torch.uint8, device="cuda")
        compact.copy_(torch.from_numpy(host.reshape(-1)).to("cuda"))
        dcounts = torch.zeros(256, dtype=torch.int64, device="cuda")
        dT = torch.zeros(1, dtype=torch.int32, device="cuda")
        hk = []
        for i in range(3 + 10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dcounts.fill_(-1)
            dT.fill_(-2)
            a.record(stream)
            _lib.call("vx_histogram_otsu_device", C.c_void_p(compact.data_ptr()), nvox,
                      C.c_void_p(dcounts.data_ptr()), C.c_void_p(dT.data_ptr()), sptr)
            b.record(stream)
            torch.cuda.synchronize()
            if i >= 3:
                hk.append(a.elapsed_time(b))
        got = dcounts.cpu().numpy()
        if not (np.array_equal(got, counts) and int(dT.item()) == hist.otsu_threshold):
            raise SystemExit(f"K1/K2 mismatch: T {int(dT.item())} vs {hist.otsu_threshold}, "
                             f"{int((got != counts).sum())} bins differ")
        hms = statistics.median(hk)
        peak, peak_kind = peaks()
        gbs = nvox / (hms * 1e-3) / 1e9
        hist_line = {"value": gbs, "unit": "GB/s", "ms": hms, "bytes": nvox,
                     "frac": gbs / peak, "peak": peak, "otsu_T": hist.otsu_threshold,
                     "kernels": "hist_otsu_kernel (K1+K2 fused, one launch, last block runs Otsu), median of 10, L2 flushed"}
        del compact

    # ---- e2e through the drop-in API ----
    e2e = None
    if rank == 0 and world == 1 and not args.no_e2e:
        for _ in range(3):
            vx.render_frame(volume, cam, params, cfg, hist)
        e2e_t = []
        for _ in range(args.steps):
            flush.zero_()  # L2 flushed between frames, outside the timed call
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = vx.render_frame(volume, cam, params, cfg, hist)
            e2e_t.append(time.perf_counter() - t0)
        e2e_s = sum(e2e_t) / len(e2e_t)
        h2d = C.sizeof(_lib.vx_ray_setup) + C.sizeof(_lib.vx_render_params) + C.sizeof(
            _lib.vx_filter_config)
        e2e = {"value": 1.0 / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": W * H + 259 * 8,
               "ms_median": statistics.median(e2e_t) * 1e3,
               "ms_max": max(e2e_t) * 1e3,
               "api": "paper_1807_03119_b200.render_frame -> Frame(pixels: host numpy)"}
        assert np.array_equal(f.pixels.reshape(-1), pixels.cpu().numpy())

    # ---- roofline of the dominant kernel ----
    peak, peak_kind = peaks()
    kms = statistics.mean(kern_ms)
    alg_bytes = nvox + W * H  # volume read once + frame written
    achieved = alg_bytes / (kms * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("raycast_dram_bytes")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as orc

        cv = orc.cam_vector(cam.position, cam.look_at, W, H)
        cpu = cpu_baseline(host, cv, W, H, args.filter, float(cfg.threshold), hist,
                           args.cpu_rows, 1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": f"insect_{args.size}^3 (C2 recipe x{args.size / 512:g}) @ "
                                   f"{W}x{H}, {args.filter}, Otsu T={hist.otsu_threshold}",
                       "volume": [args.size] * 3, "image": [W, H], "filter": args.filter,
                       "parallelism": f"sort-first tiles x{world}" if world > 1 else "single",
                       "l2": "flushed (256 MiB write) between steps, outside the step events",
                       "skip": not args.no_skip, "phantom_gen_s": round(gen_s, 2)},
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "raycast_kernel<LOCAL_CLUSTER>", "kernel_ms": kms,
                         "alg_bytes": alg_bytes, "peak_source": peak_kind,
                         "dram_achieved": (traffic / (kms * 1e-3) / 1e9) if traffic else None,
                         "dram_frac": (traffic / (kms * 1e-3) / 1e9 / peak) if traffic else None,
                         "note": "effective: exact empty-space skipping reads far less than the "
                                 "volume (frac > 1 = faster than reading it once); traffic = ncu "
                                 "dram bytes per launch, dram_frac = that traffic's share of the "
                                 "peak (the kernel is latency/issue-bound, not HBM-bound)"},
            "otsu_hist": hist_line,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "frame": {"hits": hit_count, "samples": samples, "trunc_flag": trunc_flag,
                      "kernel_ms_median": statistics.median(kern_ms),
                      "step_ms_median": statistics.median(step_ms),
                      "cold_ms": cold_ms,
                      "cold_note": "wall ms of warm-up frames 1-2: frame 1 renders on the "
                                   "candidate distance map (built with the volume) and schedules "
                                   "its first tile order, frame 2 builds the filter's "
                                   "accepted-cell map; timed frames reuse both (per "
                                   "volume/setting caches)"},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
