#!/usr/bin/env bash
# Build recipe for oracle/_ref: the UNMODIFIED reference package (gnncache 0.1.0, pure
# Python/numpy) installed from /root/reference into oracle/_ref, exactly as pip builds
# it. Test/bench infrastructure only: bench.py --impl reference and the cpu_baseline
# leg time it, tests compare against it. oracle/_ref is git-ignored (it is a build
# output, not source in this repo) but not gpurun-ignored, so it travels to the GPU box
# like the built .so. /root/reference is read-only: the build runs from a copy in /tmp.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${GC_REFERENCE_PKG:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -f "$SRC/pyproject.toml" ]; then
    echo "build_ref: $SRC not found; oracle/_ref not rebuilt" >&2
    exit 0
fi
TMP="$(mktemp -d /tmp/gc_refbuild.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT.tmp"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$OUT.tmp" "$TMP/pkg"
rm -rf "$OUT"
mv "$OUT.tmp" "$OUT"
echo "build_ref: reference installed into $OUT"
