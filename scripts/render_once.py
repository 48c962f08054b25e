"""Render a config a few times through vx_render_device (profiling target)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
from scripts.config_sweep import frame_runner
from paper_1807_03119_b200 import phantoms
from paper_1807_03119_b200.histogram import model_from_counts
from paper_1807_03119_b200.volume import generate_phantom_device

n = int(sys.argv[1]); kind = sys.argv[2]; W = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
dvol = generate_phantom_device(phantoms.insect_phantom_spec(n))
hist = model_from_counts(dvol.counts())
run, small = frame_runner(dvol, hist, W, kind, stream)
for _ in range(4):
    run()
torch.cuda.synchronize()
print("ok", small.cpu().numpy()[256:258])
