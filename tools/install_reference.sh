#!/usr/bin/env bash
# Installs the UNMODIFIED reference (halftile, pure Python) into baseline/_ref
# -- git-ignored, but it travels to the GPU box with gpurun -- plus a copy of
# its own test suite (baseline/_ref/halftile_tests) for
# tools/run_reference_tests.py.  Run here (the box has no /root/reference).
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/root/reference/pkg
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"   # the build writes into the source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/halftile_tests"
rm -rf "$TMP"
echo "installed halftile $(python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import halftile; print(halftile.__version__)") into baseline/_ref"
