#!/usr/bin/env bash
# Stage the UNMODIFIED reference package into the git-ignored baseline/_ref
# (offline wheelhouse, no index).  The directory travels to the GPU box with
# the gpurun snapshot, where tests/test_gpu_reference_engine.py imports it.
# /root/reference is read-only, so the build runs from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
echo "staged: $(ls "$ROOT/baseline/_ref")"
