#!/bin/bash
# baseline/install_reference.sh -- installs the UNMODIFIED reference package (dhsa, with its own
# compiled extension dhsa._core) from /root/reference/pkg into baseline/_ref/ (git-ignored, not
# gpurun-ignored: it travels to the GPU box with the snapshot).  Nothing from the reference enters
# the repository's history.  The build writes generated C next to the .pyx, and /root/reference is
# read-only, so it runs from a throw-away copy under /tmp.  No-op when /root/reference is absent
# (GPU box: the installed copy that travelled with the repo is used).
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=${REFERENCE_PKG:-/root/reference/pkg}
if [ ! -d "$SRC" ]; then
  echo "reference sources absent: keeping baseline/_ref as it is"
  exit 0
fi
TMP=$(mktemp -d /tmp/dhsa_ref_build.XXXXXX)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg"
# the reference's own test files travel too (git-ignored like _ref): tests/test_gpu_reference_suite.py
# runs them, unmodified, against the CUDA sketch on the GPU box
rm -rf "$HERE/_ref_tests"
mkdir -p "$HERE/_ref_tests"
cp "$SRC"/tests/*.py "$HERE/_ref_tests/"
rm -rf "$TMP"
python - <<PY
import sys
sys.path.insert(0, "$HERE/_ref")
import dhsa
from dhsa._kernels import available_backends
print("installed dhsa", dhsa.__file__, "backends", available_backends())
assert "compiled" in available_backends(), "the reference's compiled extension did not build"
PY
