"""One fused K1+K2 over an edge^3 random uint8 volume (profiling target)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1807_03119_b200 import _lib

edge = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = edge ** 3
t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
counts = torch.zeros(257, dtype=torch.int64, device="cuda")
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    _lib.call("vx_histogram_otsu_device", C.c_void_p(t.data_ptr()), n, C.c_void_p(counts.data_ptr()),
              C.c_void_p(counts.data_ptr() + 2048), sp)
torch.cuda.synchronize()
print("ok", int(counts[:256].sum()))
