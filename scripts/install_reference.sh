#!/usr/bin/env bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored, travels
# to the GPU box with gpurun) and place its own test suite next to it, so the
# drop-in test (tests/test_dropin_reference_suite.py) can run the reference's tests
# on the GPU context.  /root/reference is read-only: build from a copy in /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/cryptogen_tests"
cp -r "$SRC/configs" "$ROOT/baseline/_ref/configs"
rm -rf "$TMP"
echo "installed cryptogen into $ROOT/baseline/_ref (+ cryptogen_tests/)"
