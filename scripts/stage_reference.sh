#!/usr/bin/env bash
# Stage the UNMODIFIED reference package (rafem 0.1.0) into baseline/_ref.
#
# baseline/_ref is git-ignored but travels to the GPU box with gpurun and the
# driver's snapshot, so the reference's own run_simulation, its test suite
# and the --impl reference bench arm can run there (the box has no
# /root/reference).  Nothing under /root/reference is written: the package
# is installed from a copy under /tmp.  Its tests go to
# baseline/_ref/rafem_tests (run with tests/seam_plugin.py, see
# tests/test_gpu_reference_seam.py).
#
#   scripts/stage_reference.sh [/root/reference/pkg]
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
if [ ! -d "$SRC/src/rafem" ]; then
    echo "stage_reference: no reference package at $SRC (nothing staged)"
    exit 0
fi
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
# matplotlib (plots only) is not in the image: --no-deps
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/rafem_tests"
echo "stage_reference: rafem $(python -c 'import sys; sys.path.insert(0, sys.argv[1]); import rafem, importlib.metadata as m; print(m.version("rafem"))' "$ROOT/baseline/_ref" 2>/dev/null || echo '?') staged in baseline/_ref"
