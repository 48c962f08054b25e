"""Debug build (-DVX_HIST_TIMING): %globaltimer marks inside the fused K1+K2
kernel's last block (ns from the last block passing its ticket)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1807_03119_b200 import _lib

lib = _lib.load()
for edge in (256, 512, 1024):
    n = edge ** 3
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    counts = torch.zeros(257, dtype=torch.int64, device="cuda")
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(5):
        _lib.call("vx_histogram_otsu_device", C.c_void_p(t.data_ptr()), n,
                  C.c_void_p(counts.data_ptr()), C.c_void_p(counts.data_ptr() + 2048), sp)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 8)()
    lib.vx_debug_hist_times(buf)
    t0 = buf[7]
    print(edge, {"loads_done": buf[4] - t0, "scan_local": buf[6] - t0, "scan_synced": buf[0] - t0,
                 "screen1": buf[1] - t0, "screen2": buf[2] - t0, "exact": buf[3] - t0,
                 "end": buf[5] - t0})
