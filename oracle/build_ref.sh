#!/usr/bin/env bash
# Recipe for oracle/_ref: installs the UNMODIFIED reference package (`helmfft`,
# pure Python on numpy/scipy) from /root/reference into oracle/_ref, so that
# the CPU reference arm of bench.py and the reference-facing tests can import
# the stock code on the GPU box (where /root/reference does not exist).
# Test and baseline infrastructure only: the product never imports it.
# The build copies the source to /tmp first (/root/reference is read-only);
# nothing of the reference lands in git (oracle/_ref/ is git-ignored).
set -euo pipefail
SRC=${1:-/root/reference/pkg}
HERE="$(cd "$(dirname "$0")" && pwd)"
[ -d "$SRC" ] || { echo "build_ref: $SRC absent; keeping oracle/_ref as is"; exit 0; }
TMP=$(mktemp -d /tmp/helmfft_ref.XXXXXX)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --target "$HERE/_ref" "$TMP/pkg"
echo "build_ref: installed $(ls "$HERE/_ref" | tr '\n' ' ')into $HERE/_ref"
