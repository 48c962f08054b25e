#!/usr/bin/env python
"""Headline benchmark: filtered frames/s at 1024^2 on a 1024^3 CT volume (B200),
plus the Otsu histogram throughput against HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

``--gpus N`` without a torchrun environment launches N ranks itself
(torch.distributed.run on 127.0.0.1).  With fewer GPUs than ranks the ranks
share GPUs (functional mode: gloo for set-up, host-ordered frames; its
timings are not a scaling number and say so).

Workload (BASELINE.json metric): the CT-like insect phantom
(C2 recipe scaled to 1024^3, generated on the device by K7), Otsu threshold
from the device histogram (K1 + K2), orbit camera defaults, 1024x1024 image,
local-cluster filter (M=3, d=1), Sobel + Phong.  A step is one full frame.

value      frames/s with the volume resident in HBM; per-step CUDA events on
           the launch stream around the frame (N>1: every rank's K4 writing
           its tiles into rank 0's frame, rank 0's wait for all ranks' flags
           and the slot release); L2 flushed (256 MiB write) between steps,
           outside the events; total time = max over ranks.
e2e        the same frames through the public drop-in API with host outputs
           (N=1: render_frame; N>1: distributed.render_sharded on every rank,
           rank 0's wall clock): camera / params uploaded and the 1 MiB frame
           + histogram read back each step.
e2e_orbit  N=1: 100 frames through render_frame with the camera moving 1
           degree of azimuth per frame (the paper's interactive case).
roofline   dominant kernel (K4 raycast): SURVEY §8d algorithmic bytes
           (N voxels + W*H) / kernel time vs MEASURED_PEAKS hbm_gbs, labelled
           "effective" (skipping reads far less); dram_* from an ncu pass of
           this same workload run by this script (cold cache per launch), for
           the skipping kernel and a full-traversal (no-skip) kernel.
cpu_baseline  oracle/ C restatement of the reference (1 thread) on a bounded
           row sample of the same frame, extrapolated to frames/s.
"""

from __future__ import annotations

import argparse
import ctypes as C
import csv
import hashlib
import io
import json
import os
import shutil
import socket
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


def workload_name(size: int, image: int, filt: str, u16: bool = False) -> str:
    """The config.workload string both arms print (identical for one config)."""
    src = "uint16 CT file" if u16 else "uint8"
    return (f"insect_{size}^3 (C2 recipe x{size / 512:g}, {src}) @ "
            f"{image}x{image}, {filt}, Otsu T")


def parse(argv=None):
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
    ap.add_argument("--orbit", type=int, default=100, help="orbit leg frames (0: off)")
    ap.add_argument("--noskip-steps", type=int, default=5, help="full-traversal leg frames")
    ap.add_argument("--ncu", default="auto", choices=["auto", "on", "off"],
                    help="DRAM traffic pass under ncu (auto: when ncu is on PATH and N=1)")
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-python-ref", dest="python_ref", action="store_false",
                    help="reference arm: skip timing the Python reference at C2")
    ap.add_argument("--u16", action="store_true",
                    help="C4 input: write the phantom as a 16-bit CT file and ingest it "
                         "through load_raw (rank 0), instead of generating it in HBM")
    ap.add_argument("--sync", default="auto", choices=["auto", "device", "host"],
                    help="N>1 frame ordering (auto: device flags unless ranks share a GPU)")
    return ap.parse_args(argv)


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


def sha16(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


# ------------------------------------------------------------------------------------


def python_reference_c2(threads: int) -> dict:
    """The unmodified Python reference (baseline/_ref, scripts/install_reference.sh)
    timed on this host at BASELINE.json C2 (insect 512^3 @1024^2, local
    cluster): render_frame with 1 worker and with every host thread.  A stated
    baseline beside the arm's C port of the same path."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "voxray" / "render.py").exists():
        return {"status": "baseline/_ref not installed"}
    sys.path.insert(0, str(ref))
    try:
        import voxray
        from oracle import oracle as orc

        from paper_1807_03119_b200 import phantoms  # the spec constants only (dataclasses)

        data = orc.phantom(phantoms.insect_phantom_spec(512).to_json(), threads=threads)
        vol = voxray.Volume(dims=(512, 512, 512), data=data)
        hist = voxray.build_histogram(vol)
        cam = voxray.orbit_camera(vol)
        params = voxray.RenderParams(width=1024, height=1024)
        cfg = voxray.FilterConfig(kind=voxray.FilterKind.LOCAL_CLUSTER)
        out = {"status": "ok", "config": "C2: insect_512^3 @ 1024x1024, local-cluster, Otsu T",
               "module": voxray.__file__, "otsu_T": int(hist.otsu_threshold)}
        for workers in (1, threads):
            t0 = time.perf_counter()
            f = voxray.render_frame(vol, cam, params, cfg, hist, workers=workers)
            out[f"frame_s_workers_{workers}"] = time.perf_counter() - t0
        out["frame_sha256_16"] = sha16(f.pixels)
        return out
    except Exception as exc:  # reported, never fatal for the arm
        return {"status": f"failed: {exc!r}"[:300]}
    finally:
        sys.path.remove(str(ref))


def run_reference(args):
    """--impl reference: the reference's CPU path (the oracle C restatement,
    oracle/vxoracle.c, pinned to the live reference's frames) on every host
    thread, whole frames of the same workload."""
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
    times = []
    pixels = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = orc.render(vol, cam, W, H, kind=args.filter, threshold=float(hm["otsu"]),
                       sigma_band=2.0 * hm["global_sigma"], probabilities=hm["probabilities"],
                       threads=threads, diagnostics=False)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
        pixels = r["pixels"]
    per_frame = statistics.mean(times)
    value = 1.0 / per_frame
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_frame * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": workload_name(args.size, args.image, args.filter, args.u16),
                   "volume": [args.size] * 3, "image": [W, H], "filter": args.filter,
                   "otsu_T": hm["otsu"]},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": f"whole {W}x{H} frames ({args.steps} timed after "
                                   f"{args.warmup} warm-up) on {threads} host threads; phantom "
                                   f"generated on the host in {gen_s:.1f}s"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "frame": {"sha256_16": sha16(pixels), "otsu_T": hm["otsu"]},
        "python_reference": python_reference_c2(threads) if args.python_ref else None,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------


def spawn(args) -> int:
    """--gpus N outside torchrun: launch the N ranks (one process each)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def ncu_pass(args, peak):
    """DRAM bytes and duration of K4 per launch, from one ncu run of this
    workload (--ncu-child): the warm skipping frame and a full-traversal
    frame.  Cold cache per launch (ncu's default cache control)."""
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if Path("/usr/local/cuda/bin/ncu").exists()
                                  else None)
    if ncu is None:
        return {"status": "ncu not found"}
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    log = out / "bench_ncu.csv"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:raycast_kernel", "-c", "4", "--csv",
           "--log-file", str(log), sys.executable, str(Path(__file__).resolve()), "--ncu-child",
           "--size", str(args.size), "--image", str(args.image), "--filter", args.filter]
    t0 = time.perf_counter()
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=420)
    except subprocess.TimeoutExpired:
        return {"status": "ncu timed out"}
    if res.returncode != 0 or not log.exists():
        return {"status": f"ncu rc={res.returncode}", "tail": (res.stdout + res.stderr)[-300:]}
    rows = list(csv.DictReader(io.StringIO("".join(
        l for l in log.read_text().splitlines(True) if l.startswith('"')))))
    per: dict[int, dict] = {}
    for r in rows:
        try:
            i = int(r["ID"])
            v = float(r["Metric Value"].replace(",", ""))
        except (KeyError, ValueError):
            continue
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                 "GB": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9,
                 "us": 1e-6, "ms": 1e-3}.get(unit, 1)
        per.setdefault(i, {})[r["Metric Name"]] = v * scale
    ids = sorted(per)
    if len(ids) < 4:
        return {"status": f"ncu captured {len(ids)} launches", "tail": res.stdout[-300:]}

    def leg(i):
        m = per[i]
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        t = m.get("gpu__time_duration.sum", 0.0)
        return {"dram_bytes": b, "ncu_ms": t * 1e3, "dram_gbs": b / t / 1e9 if t else None,
                "dram_frac": (b / t / 1e9 / peak) if t else None}

    return {"status": "ok", "skip": leg(ids[2]), "noskip": leg(ids[3]),
            "seconds": round(time.perf_counter() - t0, 1),
            "command": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                       "gpu__time_duration.sum -k regex:raycast_kernel -c 4 bench.py --ncu-child "
                       "(launches 3 = warm skipping frame, 4 = no-skip frame)"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1807_03119_b200 as vx
    from paper_1807_03119_b200 import _lib, distributed, phantoms
    from paper_1807_03119_b200.filters import native_config
    from paper_1807_03119_b200.histogram import model_from_counts
    from paper_1807_03119_b200.render import native_params, ray_setup
    from paper_1807_03119_b200.volume import (_attach, _phantom_args, device_volume,
                                              generate_phantom_device)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = max(1, torch.cuda.device_count())
    shared = world > ndev  # functional mode: ranks share GPUs
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    _lib.call("vx_set_device", dev_index)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
    W = H = args.image
    nvox = args.size ** 3
    spec = phantoms.insect_phantom_spec(args.size)

    # a dedicated (non-null) stream: torch work, events and our kernels share
    # it (for the C-ABI, stream 0 would be the legacy default stream)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = C.c_void_p(stream.cuda_stream)

    # ---- workload: every rank holds the full volume (sort-first) ----
    t0 = time.perf_counter()
    volume = None  # host Volume (rank 0), when the workload has one
    ingest = None
    if args.u16:
        # C4 as BASELINE.json states it: a uint16 CT file through load_raw's
        # streamed device path (volume.py:122-151) on the source rank
        if rank == 0:
            tmp = Path(os.environ.get("TMPDIR", "/tmp")) / f"vx_ct{args.size}_{os.getpid()}.raw"
            phantoms.write_ct_u16(spec, tmp)
            torch.cuda.synchronize()
            ti = time.perf_counter()
            volume = vx.load_raw(tmp)
            ingest_s = time.perf_counter() - ti
            ingest = {"file_bytes": 2 * nvox, "seconds": ingest_s,
                      "gbs": 2 * nvox / ingest_s / 1e9,
                      "path": "load_raw -> vx_volume_load_raw (pread slots overlapped with H2D, "
                              "u16 rescale on the device)"}
            tmp.unlink()
            Path(str(tmp)[:-4] + ".meta.json").unlink()
        if world == 1:
            dvol = device_volume(volume)
            counts = dvol.counts()
            hist = model_from_counts(counts)
        else:
            dvol = distributed.replicate_volume(spec.dims, volume=volume)  # NCCL broadcast
            hist = distributed.histogram_sharded(dvol)
            counts = hist.counts
    elif world == 1:
        dvol = generate_phantom_device(spec)
        counts = dvol.counts()
        hist = model_from_counts(counts)  # K1 (at creation) + K2
    else:
        table, n_shapes, seed, spots, k = _phantom_args(spec)

        def fill(t):  # K7 on the source rank, straight into the broadcast buffer
            _lib.call("vx_phantom_device", C.c_void_p(t.data_ptr()), *spec.dims,
                      _lib.ptr(table), n_shapes, float(spec.noise_sigma), seed, _lib.ptr(spots),
                      k, int(spec.spot_noise.intensity), sptr)

        dvol = distributed.replicate_volume(spec.dims, fill=fill)  # NCCL broadcast
        hist = distributed.histogram_sharded(dvol)  # z-slab K1 + all-reduce + K2
        counts = hist.counts
    if world > 1 and not np.array_equal(counts, dvol.counts()):
        raise SystemExit("sharded histogram differs from the replica's own K1")
    gen_s = time.perf_counter() - t0

    cfg = vx.FilterConfig(kind=vx.FilterKind.from_name(args.filter)).resolve_threshold(hist)
    nx, ny, nz = spec.dims
    target = ((nx - 1) / 2.0, (ny - 1) / 2.0, (nz - 1) / 2.0)
    import math

    dist_ = 2.2 * math.sqrt(nx * nx + ny * ny + nz * nz) / 2.0

    def orbit_cam(az):  # render.orbit_camera without a host Volume
        el, a = math.radians(25.0), math.radians(az)
        pos = (target[0] + dist_ * math.cos(el) * math.cos(a),
               target[1] + dist_ * math.cos(el) * math.sin(a),
               target[2] + dist_ * math.sin(el))
        return vx.Camera(position=pos, look_at=target)

    cam = orbit_cam(45.0)
    params = vx.RenderParams(width=W, height=H)
    rs = ray_setup(cam, W, H)
    rp = native_params(params, skip=not args.no_skip)
    fc = native_config(cfg, hist)

    pixels = torch.zeros(H * W, dtype=torch.uint8, device="cuda")
    small = torch.zeros(260, dtype=torch.int64, device="cuda")
    out = _lib.vx_render_out()
    out.pixels = pixels.data_ptr()
    out.image_hist = small.data_ptr()
    out.hit_count = small.data_ptr() + 256 * 8
    out.samples = small.data_ptr() + 257 * 8
    out.trunc_flag = small.data_ptr() + 258 * 8
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fg = distributed.FrameGroup(W * H, sync=args.sync) if world > 1 else None

    def frame():
        if fg is None:
            small.zero_()
            _lib.call("vx_render_device", dvol.handle, C.byref(rs), C.byref(rp), C.byref(fc),
                      None, C.byref(out), sptr)
        else:
            fg.render(dvol, rs, rp, fc, stream.cuda_stream)
            fg.finish(stream)
            fg.release(stream.cuda_stream)

    if args.ncu_child:  # frames for the ncu pass: 3 skipping (cold, map build, warm) + 1 no-skip
        for _ in range(3):
            frame()
        rp0 = native_params(params, skip=False)
        small.zero_()
        _lib.call("vx_render_device", dvol.handle, C.byref(rs), C.byref(rp0), C.byref(fc),
                  None, C.byref(out), sptr)
        torch.cuda.synchronize()
        return 0

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
    host_t0 = time.perf_counter()
    with ClockSampler(dev_index) as clocks:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            if fg is None:
                small.zero_()
                kern[i][0].record(stream)
                _lib.call("vx_render_device", dvol.handle, C.byref(rs), C.byref(rp), C.byref(fc),
                          None, C.byref(out), sptr)
                kern[i][1].record(stream)
            else:
                kern[i][0].record(stream)
                fg.render(dvol, rs, rp, fc, stream.cuda_stream)
                kern[i][1].record(stream)
                fg.finish(stream)
                fg.release(stream.cuda_stream)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    host_s = time.perf_counter() - host_t0
    launches = _lib.launches()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    kern_ms = [a.elapsed_time(b) for a, b in kern]
    total_ms = sum(step_ms)
    if fg is not None and fg.host_sync:
        # host-ordered frames: the per-frame barrier is outside the events
        total_ms = host_s * 1000.0
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = 1000.0 / ms_per_step

    # ---- the frame itself (identical for any N: per-ray pure functions) ----
    if fg is None:
        sm = small.cpu().numpy()
        trunc_flag, samples, hit_count = int(sm[258]), int(sm[257]), int(sm[256])
        frame_pixels = pixels.cpu().numpy()
    else:
        f = distributed.render_sharded(dvol, cam, params, cfg, hist, fgroup=fg)
        trunc_flag, samples = 0, None
        hit_count = f.hit_count if f is not None else None
        frame_pixels = f.pixels.reshape(-1).copy() if f is not None else None
    frame_info = {"hits": hit_count, "samples": samples, "trunc_flag": trunc_flag,
                  "sha256_16": sha16(frame_pixels) if frame_pixels is not None else None,
                  "kernel_ms_median": statistics.median(kern_ms),
                  "step_ms_median": statistics.median(step_ms), "cold_ms": cold_ms,
                  "cold_note": "wall ms of warm-up frames 1-2: frame 1 renders on the candidate "
                               "distance map (built with the volume) and schedules its first "
                               "tile order, frame 2 builds the filter's accepted-cell map; timed "
                               "frames reuse both (per volume/setting caches)"}

    # ---- march statistics of the frame: the dependent-lookup latency model ----
    lat_model = None
    if world == 1:
        diag = torch.zeros(8, dtype=torch.int64, device="cuda")
        small.zero_()
        out.diag = diag.data_ptr()
        _lib.call("vx_render_device", dvol.handle, C.byref(rs), C.byref(rp), C.byref(fc), None,
                  C.byref(out), sptr)
        torch.cuda.synchronize()
        out.diag = None
        dg = dict(zip(("lookups", "skips", "chunks_skipped", "unused", "sample_groups",
                       "filter_evals", "hits", "iterations"), diag.cpu().tolist()))
        rays = W * H
        sm_count = torch.cuda.get_device_properties(dev_index).multi_processor_count
        clk = (clocks.summary().get("sm_mhz") or 1965.0) * 1e6
        l2_cycles = 248.0  # B300_MICROARCH.md: L2 hit 234 (near die) / 262 (far die)
        warp_steps = dg["iterations"] / 32.0
        model_ms = warp_steps * l2_cycles / clk / (sm_count * 32) * 1e3
        lat_model = {
            **dg, "rays": rays,
            "iterations_per_ray": dg["iterations"] / rays,
            "lookups_per_ray": dg["lookups"] / rays,
            "samples_per_ray": samples / rays if samples else None,
            "model_ms": model_ms, "measured_kernel_ms": statistics.median(kern_ms),
            "round_trips_per_step": statistics.median(kern_ms) / model_ms if model_ms else None,
            "note": "model = (lane march steps / 32) warp-steps x one L2 round trip (248 cycles) "
                    "spread over every resident warp (SMs x 32), i.e. the frame time if every "
                    "step were a single perfectly overlapped dependent L2 access; "
                    "round_trips_per_step = measured / model"}

    # ---- e2e through the drop-in API (host frame out) ----
    e2e = None
    host = volume.data if volume is not None else None
    if world == 1 and volume is None and (not args.no_e2e or args.orbit or not args.no_cpu):
        host = dvol.read()  # the host Volume of the e2e / CPU legs (compact copy)
        volume = _attach(vx.Volume(dims=spec.dims, data=host), dvol)
    if volume is not None:
        volume.content_hash()
    if not args.no_e2e:
        if world == 1:
            for _ in range(3):
                vx.render_frame(volume, cam, params, cfg, hist)
            e2e_t = []
            for _ in range(args.steps):
                flush.zero_()  # L2 flushed between frames, outside the timed call
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                f = vx.render_frame(volume, cam, params, cfg, hist)
                e2e_t.append(time.perf_counter() - t0)
            assert np.array_equal(f.pixels.reshape(-1), frame_pixels)
            api = "paper_1807_03119_b200.render_frame -> Frame(pixels: host numpy)"
        else:
            for _ in range(3):
                distributed.render_sharded(dvol, cam, params, cfg, hist, fgroup=fg)
            e2e_t = []
            dist.barrier()
            for _ in range(args.steps):
                flush.zero_()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                f = distributed.render_sharded(dvol, cam, params, cfg, hist, fgroup=fg)
                e2e_t.append(time.perf_counter() - t0)
            if rank == 0:
                assert np.array_equal(f.pixels.reshape(-1), frame_pixels)
            api = ("paper_1807_03119_b200.distributed.render_sharded on every rank -> rank 0 "
                   "Frame(pixels: host numpy); wall clock of rank 0")
        e2e_s = sum(e2e_t) / len(e2e_t)
        h2d = C.sizeof(_lib.vx_ray_setup) + C.sizeof(_lib.vx_render_params) + C.sizeof(
            _lib.vx_filter_config)
        e2e = {"value": 1.0 / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": W * H + 259 * 8,
               "ms_median": statistics.median(e2e_t) * 1e3, "ms_max": max(e2e_t) * 1e3,
               "api": api}

    # ---- orbiting camera: 1 degree of azimuth per frame (service.py:228-238) ----
    orbit = None
    if world == 1 and args.orbit > 0:
        cams = [orbit_cam(45.0 + k) for k in range(args.orbit)]
        ot = []
        for c in cams:
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            vx.render_frame(volume, c, params, cfg, hist)
            ot.append((time.perf_counter() - t0) * 1e3)
        srt = sorted(ot)
        orbit = {"value": 1000.0 * len(ot) / sum(ot), "unit": "frames/s", "frames": len(ot),
                 "step_deg": 1.0, "ms_p50": statistics.median(ot),
                 "ms_p99": srt[min(len(srt) - 1, int(0.99 * len(srt)))], "ms_max": srt[-1],
                 "ms_first": ot[0],
                 "note": "render_frame per frame, a new Camera each frame (azimuth 45..144 deg), "
                         "host frame out; a moving camera renders in the tile order of frame "
                         "k-1's costs; the accepted-cell map is camera-independent (built once "
                         "per setting); orthant skip maps are built when the view enters a new "
                         "direction orthant (the ms_max outlier when it happens here)"}

    # ---- full traversal (no skipping): the march engine on every sample ----
    noskip = None
    if world == 1 and args.noskip_steps > 0:
        rp0 = native_params(params, skip=False)
        nk = []
        sm0 = None
        for i in range(args.noskip_steps + 1):
            flush.zero_()
            small.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _lib.call("vx_render_device", dvol.handle, C.byref(rs), C.byref(rp0), C.byref(fc),
                      None, C.byref(out), sptr)
            b.record(stream)
            torch.cuda.synchronize()
            if i:
                nk.append(a.elapsed_time(b))
            sm0 = small.cpu().numpy()
        if not np.array_equal(pixels.cpu().numpy(), frame_pixels):
            raise SystemExit("no-skip frame differs from the skipping frame")
        ns_ms = statistics.median(nk)
        noskip = {"kernel_ms": ns_ms, "samples": int(sm0[257]),
                  "samples_per_s": int(sm0[257]) / (ns_ms * 1e-3),
                  "frames_per_s": 1000.0 / ns_ms,
                  "note": "K4 with skipping off: every sample of every ray loaded (the "
                          "reference's march), same frame bit for bit"}

    # ---- Otsu histogram K1 over the compact 1 GiB volume (second half of the metric) ----
    hist_line = None
    if rank == 0:
        compact = torch.empty(nvox, dtype=torch.uint8, device="cuda")
        if host is not None:
            compact.copy_(torch.from_numpy(np.ascontiguousarray(host).reshape(-1)))
        else:
            table, n_shapes, seed, spots, k = _phantom_args(spec)
            _lib.call("vx_phantom_device", C.c_void_p(compact.data_ptr()), *spec.dims,
                      _lib.ptr(table), n_shapes, float(spec.noise_sigma), seed, _lib.ptr(spots),
                      k, int(spec.spot_noise.intensity), sptr)
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
                     "kernels": "hist_otsu_kernel (K1+K2 fused, one launch; an extra block "
                                "runs Otsu once every counting block is in), median of 10, "
                                "L2 flushed"}
        del compact

    # ---- roofline of the dominant kernel ----
    peak, peak_kind = peaks()
    kms = statistics.mean(kern_ms)
    alg_bytes = nvox + W * H  # volume read once + frame written
    achieved = alg_bytes / (kms * 1e-3) / 1e9
    prof = None
    run_ncu = args.ncu == "on" or (args.ncu == "auto" and world == 1 and not args.no_skip)
    if rank == 0 and world == 1 and run_ncu:
        del flush
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        prof = ncu_pass(args, peak)
    traffic = prof["skip"]["dram_bytes"] if prof and prof.get("status") == "ok" else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": f"raycast_kernel<{args.filter}>", "kernel_ms": kms,
                "alg_bytes": alg_bytes, "peak_source": peak_kind,
                "frac_kind": "effective: SURVEY §8d algorithmic bytes (volume read once + frame) "
                             "over the event-timed kernel; exact skipping reads far less, so > 1 "
                             "means faster than reading the volume once",
                "dram_achieved": (traffic / (kms * 1e-3) / 1e9) if traffic else None,
                "dram_frac": (traffic / (kms * 1e-3) / 1e9 / peak) if traffic else None,
                "dram_note": "traffic = dram__bytes_read+write of the warm skipping K4 launch "
                             "from this run's ncu pass (cold cache); dram_frac = that traffic "
                             "over the event-timed kernel vs the measured peak",
                "ncu": prof}
    if noskip is not None and prof and prof.get("status") == "ok":
        nb = prof["noskip"]["dram_bytes"]
        noskip.update({"dram_bytes": nb, "dram_gbs": nb / (noskip["kernel_ms"] * 1e-3) / 1e9,
                       "dram_frac": nb / (noskip["kernel_ms"] * 1e-3) / 1e9 / peak,
                       "alg_frac": alg_bytes / (noskip["kernel_ms"] * 1e-3) / 1e9 / peak})
    roofline["noskip"] = noskip

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as orc

        cv = orc.cam_vector(cam.position, cam.look_at, W, H)
        cpu = cpu_baseline(host, cv, W, H, args.filter, float(cfg.threshold), hist,
                           args.cpu_rows, 1)

    if rank == 0:
        if world == 1:
            par = "single"
        elif fg.host_sync:
            par = (f"sort-first tiles x{world}, ranks sharing {ndev} GPU(s): functional mode "
                   f"(gloo set-up, host-ordered frames; not a scaling number)")
        else:
            par = f"sort-first tiles x{world} (peer stores into rank 0's frame, device flags)"
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (device-generated phantom)",
            "config": {"workload": workload_name(args.size, args.image, args.filter, args.u16),
                       "volume": [args.size] * 3, "image": [W, H], "filter": args.filter,
                       "otsu_T": hist.otsu_threshold, "parallelism": par,
                       "l2": "flushed (256 MiB write) between steps, outside the step events",
                       "skip": not args.no_skip, "phantom_gen_s": round(gen_s, 2),
                       "input": ("uint16 CT file via load_raw" if args.u16
                                 else "uint8 phantom generated in HBM"),
                       "ingest": ingest},
            "e2e": e2e,
            "e2e_orbit": orbit,
            "gpu_launches": launches,
            "roofline": roofline,
            "latency_model": lat_model,
            "otsu_hist": hist_line,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "frame": frame_info,
        }
        print(json.dumps(line), flush=True)
    if fg is not None:
        dist.barrier()
        fg.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
