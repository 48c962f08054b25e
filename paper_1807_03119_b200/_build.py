"""Build libvoxb200.so (sm_100a) in-tree with nvcc.

Usage: python -m paper_1807_03119_b200._build [--verbose]
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libvoxb200.so"
# bounds-checked, schedule-jittered variant (tests/test_gpu_checked.py; the
# stand-in for compute-sanitizer, which is closed on this pool)
CHECKED_LIB = PKG / "libvoxb200_checked.so"
INCLUDE = PKG.parent / "include"

SOURCES = ["vx_api.cu", "vx_hist.cu", "vx_volume.cu", "vx_render.cu", "vx_io.cu", "vx_group.cu", "vx_multi.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # the exact-arithmetic contract forbids FMA contraction of the march and
    # the FP64 ray setup / shading (render.py computes with separate roundings)
    "-fmad=false",
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    "-cudart", "static",
    "-shared",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def needs_build(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    mtime = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > mtime for p in deps)


def build(verbose: bool = False, force: bool = False, checked: bool = False) -> Path:
    lib = CHECKED_LIB if checked else LIB
    if not force and not needs_build(lib):
        return lib
    cmd = [nvcc(), *NVCC_FLAGS, "-I", str(INCLUDE)]
    if checked:
        cmd += ["-DVX_DEBUG_CHECKS", "-DVX_DEBUG_JITTER"]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += [str(CSRC / s) for s in SOURCES] + ["-o", str(lib) + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        sys.stderr.write(res.stdout + res.stderr)
    os.replace(str(lib) + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True, checked="--checked" in sys.argv))
