"""Build a tuning variant of the library next to the real one.

    python scripts/build_variant.py <suffix> -DNAME=VALUE ...
    -> paper_1807_03119_b200/libvoxb200_<suffix>.so  (select with VOXB200_LIB)
"""
import subprocess
import sys

sys.path.insert(0, ".")
from paper_1807_03119_b200 import _build as b  # noqa: E402

suffix, defs = sys.argv[1], sys.argv[2:]
out = b.PKG / f"libvoxb200_{suffix}.so"
cmd = [b.nvcc(), *b.NVCC_FLAGS, "-I", str(b.INCLUDE), *defs,
       *[str(b.CSRC / s) for s in b.SOURCES], "-o", str(out)]
subprocess.run(cmd, check=True)
print(out)
