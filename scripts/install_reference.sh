#!/bin/bash
# Install the unmodified reference (voxray) into baseline/_ref, plus a copy of
# its own test-suite (baseline/_ref/tests).  baseline/_ref is git-ignored but
# travels to the GPU box with the gpurun snapshot, where
# tests/test_reference_suite.py runs the reference's tests against the
# drop-in (tests/ref_shim.py).  Needs /root/reference (build container only).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
rm -rf /tmp/voxray_refbuild
cp -r "$SRC" /tmp/voxray_refbuild          # the build writes into its source tree
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" /tmp/voxray_refbuild
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
rm -rf /tmp/voxray_refbuild
echo "installed: $(ls "$ROOT/baseline/_ref")"
