#!/usr/bin/env bash
# Install the unmodified reference (headfem) into baseline/_ref, the one offline
# install the task allows, and copy its own test suite next to it so the GPU box
# (which has no /root/reference) can run that suite with the engine patched in
# (tests/test_gpu_reference_suite.py).  baseline/_ref is git-ignored but travels
# with gpurun snapshots.
#
#   bash tools/install_reference.sh
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
DST="$ROOT/baseline/_ref"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"            # the build writes into its source tree; /root/reference is read-only
rm -rf "$DST"
# dependency resolution is the only failure mode offline (numpy/scipy are in the image): --no-deps
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DST" "$TMP/pkg"
cp -r "$SRC/tests" "$DST/headfem_tests"
rm -rf "$DST/headfem_tests/__pycache__"
python - "$DST" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import headfem, os
print("installed", headfem.__file__, "tests:", sorted(os.listdir(os.path.join(sys.argv[1], "headfem_tests"))))
PY
