#!/bin/sh
# Install the UNMODIFIED reference package (`hrt`, /root/reference/pkg) into
# baseline/_ref (git-ignored; it travels to the GPU box with the snapshot).
# Test infrastructure for tests/test_reference_dropin_gpu.py: the reference's
# own run_jacobi3d / run_pingpong driven through integration/hrt_b200_plugin.py.
# The build writes into its source tree, so it installs from a copy in /tmp.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${REFERENCE_PKG:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --no-deps --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
echo "reference installed into $ROOT/baseline/_ref"
