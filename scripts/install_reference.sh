#!/usr/bin/env bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot) and place its own test
# suite + configs beside it in baseline/_ref/picmc_suite/, so the -m gpu test
# tests/test_reference_suite_gpu.py can run the reference's tests against the
# cuda backend on a box where /root/reference does not exist.
#
# Nothing here is committed: baseline/_ref/ is in .gitignore.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
DST="$ROOT/baseline/_ref"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"          # the build writes into its source tree
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$DST" --upgrade "$TMP/pkg" >/dev/null
rm -rf "$DST/picmc_suite"
mkdir -p "$DST/picmc_suite"
cp -r "$SRC/tests" "$DST/picmc_suite/tests"
cp -r "$SRC/configs" "$DST/picmc_suite/configs"
echo "reference installed into $DST (suite in $DST/picmc_suite)"
