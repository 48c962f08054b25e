"""The bounds-checked, schedule-jittered build (libvoxb200_checked.so,
-DVX_DEBUG_CHECKS -DVX_DEBUG_JITTER) on small cases, compared with the CPU
oracle.  compute-sanitizer is closed on this GPU pool (runs under it left
GPUs needing a reset), so this is the memory / race evidence instead:

* every voxel read is checked against the zero apron (|overshoot| <= VX_PAD)
  and the padded allocation, every skip-map read against its map, every
  warp-scratch index against its array, every pixel write against the frame
  (a violation traps, the process fails);
* lanes sleep 0-2 us at random before every march step, so a missing
  __syncwarp around the warp-shared scratch (candidate lists, pass flags,
  needy-lane table) would show as a wrong frame.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

CHECKED = ROOT / "paper_1807_03119_b200" / "libvoxb200_checked.so"


def _run(args, timeout=1200):
    if not CHECKED.exists():
        from paper_1807_03119_b200 import _build

        _build.build(checked=True)
    env = dict(os.environ, VOXB200_LIB=str(CHECKED), VOXB200_NO_BUILD="1",
               PYTHONPATH=str(ROOT))
    return subprocess.run([sys.executable, *args], capture_output=True, text=True, cwd=str(ROOT),
                          env=env, timeout=timeout)


def test_checked_build_sanitize_target():
    """Every kernel family (K1-K8, split rays, tile order, frame group) on a
    48^3 phantom: no check fires and every output equals the oracle."""
    res = _run(["scripts/sanitize_target.py"])
    assert res.returncode == 0 and "sanitize target: OK" in res.stdout, \
        res.stdout[-3000:] + res.stderr[-3000:]
    assert "VX_DCHECK" not in res.stdout + res.stderr


def test_checked_build_render_and_filter_suites():
    """The GPU render / filter / acceptance parity tests under the checked build."""
    res = _run(["-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                "tests/test_gpu_render.py", "tests/test_gpu_filters.py",
                "tests/test_gpu_acceptance.py", "tests/test_gpu_volume.py"])
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    assert "VX_DCHECK" not in res.stdout + res.stderr
