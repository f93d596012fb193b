#!/usr/bin/env bash
# Install the UNMODIFIED reference (staircase, with its compiled _evalcy
# engine) into baseline/_ref.  /root/reference is read-only and its build
# writes into the source tree, so the install runs from a scratch copy.
# baseline/_ref is git-ignored but travels to the GPU box with gpurun.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
if [ ! -d "$SRC" ]; then
  echo "reference sources not found at $SRC" >&2
  exit 1
fi
TMP="$(mktemp -d /tmp/staircase_src.XXXXXX)"
cp -r "$SRC"/. "$TMP"/
chmod -R u+w "$TMP"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
  --target "$HERE/_ref" "$TMP" >"$HERE/install_ref.log" 2>&1
rm -rf "$TMP"
test -f "$HERE"/_ref/staircase/interp/_evalcy*.so
echo "installed reference into $HERE/_ref"
