#!/usr/bin/env bash
# Stage the UNMODIFIED reference under baseline/_ref (git-ignored, travels to
# the GPU box with gpurun): the `zeitlin` package installed from the wheel
# build of /root/reference/pkg (the reference arm of bench.py and the
# reference-suite run), and the reference's own pytest files in
# baseline/_ref/zeitlin_tests (run unmodified against the drop-in by
# tests/test_reference_suite_gpu.py through tools/zt_ref_plugin.py).
# Needs /root/reference (this build container only).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${1:-/root/reference}"
TMP="$(mktemp -d)"
cp -r "$REF/pkg" "$TMP/pkg"   # the build writes into its source tree
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --upgrade --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
rm -rf "$ROOT/baseline/_ref/zeitlin_tests"
cp -r "$REF/pkg/tests" "$ROOT/baseline/_ref/zeitlin_tests"
rm -rf "$TMP"
echo "staged: $(ls "$ROOT/baseline/_ref")"
