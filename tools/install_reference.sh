#!/usr/bin/env bash
# Install the UNMODIFIED reference (boardbatch, /root/reference/pkg) into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot), plus a copy of its own test suite under
# baseline/_ref/_tests for the hook-in run (tests/test_gpu_reference_hookin.py). The reference tree
# is read-only, so pip builds from a copy under /tmp. numpy is already in the image (--no-deps).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/_tests"
rm -rf "$TMP"
echo "installed: $(ls "$ROOT/baseline/_ref")"
