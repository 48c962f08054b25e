"""Histogram micro-timings: fused K1+K2 vs K1 alone vs the Otsu tail (n=0),
L2 flushed or warm, per size (CUDA events on the launch stream)."""
import ctypes as C, json, os, statistics, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1807_03119_b200 import _lib

_lib.load()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
sp = C.c_void_p(stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
counts = torch.zeros(257, dtype=torch.int64, device="cuda")
dT = counts[256:].view(torch.int32)


def timed(fn, reps=20, do_flush=True):
    out = []
    for i in range(reps + 3):
        if do_flush:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            out.append(a.elapsed_time(b) * 1e3)
    return round(statistics.median(out), 2)


res = {}
for edge in [int(e) for e in (sys.argv[1:] or ["256", "512", "1024"])]:
    n = edge ** 3
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    fused = lambda: _lib.call("vx_histogram_otsu_device", C.c_void_p(t.data_ptr()), n,
                              C.c_void_p(counts.data_ptr()), C.c_void_p(dT.data_ptr()), sp)
    k1 = lambda: _lib.call("vx_histogram_device", C.c_void_p(t.data_ptr()), n,
                           C.c_void_p(counts.data_ptr()), sp)
    empty = lambda: _lib.call("vx_histogram_otsu_device", C.c_void_p(t.data_ptr()), 0,
                              C.c_void_p(counts.data_ptr()), C.c_void_p(dT.data_ptr()), sp)
    res[f"{edge}^3"] = {"fused_flushed_us": timed(fused), "fused_warm_us": timed(fused, do_flush=False),
                        "k1_flushed_us": timed(k1), "k1_warm_us": timed(k1, do_flush=False),
                        "otsu_tail_n0_us": timed(empty, do_flush=False)}
    del t
print(json.dumps(res, indent=1))
