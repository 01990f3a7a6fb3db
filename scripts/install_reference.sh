#!/bin/sh
# Offline install of the unmodified reference package into baseline/_ref
# (git-ignored, not gpurun-ignored: it travels to the GPU box).  Used by
# tests/test_gpu_registry.py (the drop-in through popcorn's own registry).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"   # the reference tree is read-only; the build writes next to it
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
