"""The C-ABI library loads and exports every symbol include/voxb200.h declares
(CPU only: no compute calls), and the ctypes struct layouts match the C
header's (checked with a gcc-compiled probe)."""

from __future__ import annotations

import ctypes as C
import re
import shutil
import subprocess

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "voxb200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vx_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_exports_all_symbols():
    from paper_1807_03119_b200 import _lib

    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # every declared function has a ctypes signature in the binding
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)
    assert lib.vx_version() == 1


def test_binary_targets_sm100a():
    from paper_1807_03119_b200 import _lib

    if shutil.which("cuobjdump") is None and not (ROOT / "x").exists():
        cob = "/usr/local/cuda/bin/cuobjdump"
    else:
        cob = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cob, "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


STRUCTS = ["vx_ray_setup", "vx_render_params", "vx_filter_config", "vx_partition", "vx_render_out",
           "vx_group_frame"]


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc missing")
def test_struct_layouts_match_header(tmp_path):
    from paper_1807_03119_b200 import _lib

    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for s in STRUCTS:
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for fname, _ in getattr(_lib, s)._fields_:
            lines.append(f'printf("{s}.{fname} %zu\\n", offsetof({s}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                  check=True).stdout.splitlines())
    for s in STRUCTS:
        cls = getattr(_lib, s)
        assert int(got[s]) == C.sizeof(cls), s
        for fname, _ in cls._fields_:
            assert int(got[f"{s}.{fname}"]) == getattr(cls, fname).offset, (s, fname)


def test_no_device_fails_loudly(monkeypatch):
    """Without a visible GPU the product raises instead of falling back."""
    from paper_1807_03119_b200 import _lib

    lib = _lib.load()
    n = C.c_int(-1)
    rc = lib.vx_device_count(C.byref(n))
    if rc == 0 and n.value > 0:
        pytest.skip("a CUDA device is visible")
    monkeypatch.setattr(_lib, "_device_ok", None)
    with pytest.raises(_lib.NativeError, match="no CUDA device"):
        _lib.require_device()


def test_group_blob_size_matches_header():
    from paper_1807_03119_b200 import _lib

    m = re.search(r"#define VX_GROUP_BLOB_BYTES (\d+)", HEADER.read_text())
    assert m and int(m.group(1)) == _lib.VX_GROUP_BLOB_BYTES
    enum = dict(re.findall(r"(VX_GROUP_SYNC_[A-Z]+) = (-?\d+)", HEADER.read_text()))
    assert int(enum["VX_GROUP_SYNC_AUTO"]) == _lib.VX_GROUP_SYNC_AUTO
    assert int(enum["VX_GROUP_SYNC_DEVICE"]) == _lib.VX_GROUP_SYNC_DEVICE
    assert int(enum["VX_GROUP_SYNC_HOST"]) == _lib.VX_GROUP_SYNC_HOST


def test_checked_variant_carries_the_checks():
    """libvoxb200_checked.so (the compute-sanitizer stand-in run by
    tests/test_gpu_checked.py) really contains the bounds traps and the
    schedule jitter; the production library contains neither."""
    from paper_1807_03119_b200 import _build

    checked = _build.build(checked=True)
    cob = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

    def sass(p):
        return subprocess.run([cob, "-sass", str(p)], capture_output=True, text=True).stdout

    def with_op(text, op):  # functions whose SASS holds op
        return {f for f, body in re.findall(r"Function : (\S+)(.*?)(?=Function :|\Z)", text, re.S)
                if op in body}

    s_checked, s_prod = sass(checked), sass(_build.LIB)
    assert s_checked.count("BPT.TRAP") > 100 and "NANOSLEEP" in s_checked
    assert "BPT.TRAP" not in s_prod
    # the only sleep in production: the histogram's tail block polling the ticket
    assert all("hist_otsu_kernel" in f for f in with_op(s_prod, "NANOSLEEP"))
    assert with_op(s_checked, "NANOSLEEP") - with_op(s_prod, "NANOSLEEP")
