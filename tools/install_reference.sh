#!/bin/bash
# Install the UNMODIFIED reference package (pixelcodec) into baseline/_ref
# (git-ignored; it travels to the GPU box with the gpurun snapshot) for
# bench.py's reference arm / cpu_baseline and the reference-suite twin test.
# Built from a copy: /root/reference is read-only and a build writes into
# its source tree. Its own test modules are copied next to it (they run
# against this package's GPU twins in tests/test_reference_suite.py).
set -e
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no /root/reference here; baseline/_ref must already exist"; exit 0; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg" >/dev/null
mkdir -p "$REPO/baseline/_ref/reference_tests"
cp "$SRC"/tests/*.py "$REPO/baseline/_ref/reference_tests/"
cp -r "$SRC"/tests/data "$REPO/baseline/_ref/reference_tests/" 2>/dev/null || true
rm -rf "$TMP"
echo "installed pixelcodec into $REPO/baseline/_ref"
