#!/usr/bin/env bash
# Installs the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot). The build writes into the
# source tree, so it runs from a copy under /tmp (/root/reference is read-only);
# --no-deps because matplotlib is absent (numpy and numba are in the image).
# DESIGN.md section 8 "Reference install".
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "no reference at $SRC" >&2; exit 1; }
TMP="$(mktemp -d /tmp/ref_pkg.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
ls "$HERE/_ref"
