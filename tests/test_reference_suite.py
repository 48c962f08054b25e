"""The reference's own test-suite (pkg/tests) run against the drop-in on the B200.

tests/ref_shim.py maps ``voxray.{volume,histogram,filters,render,metrics}``
and the package's top-level names to this repository; the tests themselves,
their oracle (``voxray.reference``, naive loop filters) and the non-hot-path
modules (``phantoms``, ``rng``, ``grid``, ``images``, ``cli``, ``service``)
are the unmodified reference, installed by scripts/install_reference.sh into
baseline/_ref (git-ignored; it travels to the GPU box).

Deselected, each for a stated reason:
"""

from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = ROOT / "baseline" / "_ref"

FILES = ["test_histogram.py", "test_filters.py", "test_render.py", "test_metrics.py",
         "test_acceptance.py", "test_volume.py", "test_rng.py", "test_cli.py", "test_service.py"]

DESELECT = {
    "test_render.py::TestRenderFrame::test_filter_at_hit_equivalence_with_reference":
        "passes a Python filter_fn (render.py:495-508); filters run inside the ray-cast kernel "
        "and the drop-in raises RenderError instead of falling back to the CPU (SURVEY.md §8b). "
        "Its claim -- frames equal the naive reference filter at every hit -- is covered by "
        "tests/test_gpu_render.py against the oracle and the frozen reference frames",
    "test_acceptance.py::test_timing_properties":
        "asserts relative wall-clock timings of the reference's CPU renderer (criterion (a): "
        "'mean' is the fastest filtered mode, because CPU frame time tracks march length); "
        "its own docstring calls (a) noise-limited ('can fail honestly on busy machines'). It "
        "passed on the B200 in the round-2 run (profiles/r2/r2_reference_suite.txt), but a "
        "wall-clock ordering between two sub-millisecond kernels is not a parity property",
}
__doc__ += "".join(f"\n* ``{k}``: {v}." for k, v in DESELECT.items())


def test_reference_suite_on_the_drop_in(request):
    tests = REF / "tests"
    if not tests.exists():
        pytest.skip("baseline/_ref not installed (scripts/install_reference.sh)")
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_shim", "-p", "no:cacheprovider",
           "--rootdir", str(REF), "-o", "addopts=", "-W", "ignore::DeprecationWarning"]
    cmd += [str(tests / f) for f in FILES if (tests / f).exists()]
    for k in DESELECT:
        cmd += ["--deselect", f"tests/{k}"]  # node ids are relative to --rootdir
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ROOT / "tests"), str(ROOT)]))
    res = subprocess.run(cmd, capture_output=True, text=True, cwd=str(REF), env=env,
                         timeout=1800)
    tail = res.stdout.strip().splitlines()[-1] if res.stdout.strip() else ""
    counts = dict((k, int(v)) for v, k in re.findall(r"(\d+) (passed|failed|error|errors|"
                                                       r"deselected|skipped)", tail))
    request.config._ref_suite = (f"reference suite (pkg/tests, {len(FILES)} files) on the "
                                 f"drop-in: {tail}")
    assert res.returncode == 0, res.stdout[-6000:] + res.stderr[-3000:]
    # the hot-path modules were the drop-in's, the tests' oracle the reference's
    assert "voxray.render -> paper_1807_03119_b200.render" in res.stdout, res.stdout[:2000]
    assert str(REF / "voxray" / "reference.py") in res.stdout, res.stdout[:2000]
    assert counts.get("passed", 0) >= 150 and counts.get("deselected", 0) == len(DESELECT), tail
