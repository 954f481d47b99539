#!/usr/bin/env bash
# Recipe: install the UNMODIFIED reference package (pure Python, numpy only)
# from the read-only reference tree into oracle/_ref/ -- the reference's own
# implementation for the CPU baseline and `bench.py --impl reference`
# (kind "reference").  oracle/_ref/ is git-ignored (never in history) but not
# gpurun-ignored, so it travels to the GPU box with the snapshot.  The
# reference's setuptools build writes into its source tree, so it is built
# from a copy under /tmp.  Nothing here runs on the GPU box.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${ATA_REFERENCE_PKG:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src/atamul" ]; then
  echo "reference package not found at $REF: oracle/_ref not built" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/atamul_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"
rm -rf "$OUT.new"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$OUT.new" "$TMP/pkg"
rm -rf "$OUT"
mv "$OUT.new" "$OUT"
echo "installed reference atamul into $OUT"
