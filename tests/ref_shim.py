"""pytest plugin: the reference's own test-suite against the drop-in.

Loaded with ``-p ref_shim`` before the reference's conftest imports
``voxray``.  It installs a ``voxray`` package whose hot-path modules --
``volume``, ``histogram``, ``filters``, ``render``, ``metrics`` (SURVEY.md
§8a) and the top-level names of ``pkg/src/voxray/__init__.py:3-43`` -- are
this repository's (the B200 path), while everything else the tests import
(``voxray.reference`` -- the reference's naive loop filters used as the
tests' oracle -- ``phantoms``, ``rng``, ``grid``, ``images``, ``cli``,
``service``) is the unmodified reference installed in baseline/_ref.  The
reference modules import the hot-path names relatively (``from .filters
import ...``), so they run on top of the drop-in too.
"""

from __future__ import annotations

import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
DROP_IN = ("volume", "histogram", "filters", "render", "metrics")


def install() -> None:
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    import paper_1807_03119_b200 as pkg
    from paper_1807_03119_b200 import _lib

    _lib.require_device()  # no CPU fallback: the suite must run on the B200 path
    mod = types.ModuleType("voxray")
    mod.__path__ = [str(REF / "voxray")]
    mod.__file__ = str(REF / "voxray" / "__init__.py")
    mod.__version__ = "0.1.0"
    for name in pkg.__all__:
        setattr(mod, name, getattr(pkg, name))
    mod.__all__ = [n for n in pkg.__all__ if n != "frame_timing"]
    sys.modules["voxray"] = mod
    for sub in DROP_IN:
        m = __import__(f"paper_1807_03119_b200.{sub}", fromlist=["_"])
        sys.modules[f"voxray.{sub}"] = m
        setattr(mod, sub, m)


install()


def pytest_report_header(config):
    import voxray
    import voxray.render

    return [f"ref_shim: voxray.render -> {voxray.render.__name__}, "
            f"voxray.reference -> {__import__('voxray.reference').reference.__file__}"]
