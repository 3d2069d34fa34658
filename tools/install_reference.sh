#!/usr/bin/env bash
# Install the unmodified reference (the `spdnn` package) into baseline/_ref
# (git-ignored; travels to the GPU box with the gpurun snapshot), and put the
# reference's own test suite next to it for tests/test_reference_suite.py.
# Run in the build container, where /root/reference exists.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"            # the build writes into the source tree
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref/tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
rm -rf "$TMP"
echo "installed spdnn + tests into $ROOT/baseline/_ref"
