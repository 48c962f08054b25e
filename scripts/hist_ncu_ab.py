"""Fused K1+K2 launches of several library variants in one process, for one
ncu launch list (gpu__time_duration per kernel, in launch order):

    ncu --metrics gpu__time_duration.sum -k regex:hist_otsu --csv \\
        python scripts/hist_ncu_ab.py lib_a.so lib_b.so ...

Per library: sizes 256^3, 512^3, 1024^3 (env HIST_SIZES), three launches each, L2 flushed
before every launch.  Prints the launch order."""
import ctypes as C
import os
import sys

import torch

libs = [C.CDLL(p) for p in sys.argv[1:]]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
counts = torch.zeros(257, dtype=torch.int64, device="cuda")
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
order = []
for edge in [int(e) for e in os.environ.get("HIST_SIZES", "256 512 1024").split()]:
    n = edge ** 3
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    for p, lib in zip(sys.argv[1:], libs):
        fn = lib.vx_histogram_otsu_device
        fn.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        for _ in range(3):
            flush.zero_()
            rc = fn(C.c_void_p(t.data_ptr()), n, C.c_void_p(counts.data_ptr()),
                    C.c_void_p(counts.data_ptr() + 2048), sp)
            assert rc == 0
            order.append(f"{p.rsplit('/', 1)[-1]} {edge}^3")
    torch.cuda.synchronize()
    del t
print("\n".join(order))
