"""Debug build (-DVX_HIST_TIMING): %globaltimer marks of the fused K1+K2
kernel, ns relative to the first block's start: last block done counting,
last block done merging, last block's ticket, Otsu phases, end."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1807_03119_b200 import _lib

lib = _lib.load()
buf = (C.c_ulonglong * 16)()
for edge in [int(e) for e in (sys.argv[1:] or ["256", "512", "1024"])]:
    n = edge ** 3
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    counts = torch.zeros(257, dtype=torch.int64, device="cuda")
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(4):
        flush.zero_()
        torch.cuda.synchronize()
        lib.vx_debug_hist_times(buf)  # reset
        _lib.call("vx_histogram_otsu_device", C.c_void_p(t.data_ptr()), n,
                  C.c_void_p(counts.data_ptr()), C.c_void_p(counts.data_ptr() + 2048), sp)
        torch.cuda.synchronize()
    lib.vx_debug_hist_times(buf)
    t0 = buf[8]
    rel = lambda k: round((buf[k] - t0) / 1e3, 2)
    print(edge, {"first_counting_done_us": rel(11), "counting_done_us": rel(9), "merged_us": rel(10), "ticket_us": rel(7),
                 "otsu_loaded_us": rel(4), "scan_us": rel(0), "screen_us": rel(2),
                 "exact_us": rel(3), "end_us": rel(5)})
