#!/usr/bin/env bash
# Install the reference planner (maniplan) into oracle/_ref/ -- the stock
# build: `pip install` of /root/reference/pkg with its own setup.py (only
# _kernels/_compiled.pyx is compiled, with the reference's flags,
# pkg/setup.py:40-61), from a scratch copy because the mount is read-only.
# The pure-Python modules are then byte-compiled in place to sourceless .pyc
# (`compileall -b`, the unmodified modules' own bytecode, suffix .refpyc) so the package
# imports on the GPU box, where /root/reference is absent, without reference
# source text landing in the working tree.  TEST / BASELINE INFRASTRUCTURE
# ONLY: the product never imports it.
set -euo pipefail
PKG=${REF_PKG:-/root/reference/pkg}
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
OUT="$HERE/_ref"
PY=${PYTHON:-python3}
[ -d "$PKG/src/maniplan" ] || { echo "reference package not found at $PKG" >&2; exit 1; }
TMP=$(mktemp -d /tmp/cprrtc_refbuild.XXXXXX)
trap 'rm -rf "$TMP"' EXIT
cp -r "$PKG" "$TMP/pkg"
find "$TMP/pkg" -name '__pycache__' -prune -exec rm -rf {} +
"$PY" -m pip install --no-index --no-build-isolation --no-deps --quiet \
    --target "$TMP/site" "$TMP/pkg" > "$TMP/pip.log" 2>&1 || { tail -30 "$TMP/pip.log"; exit 1; }
ls "$TMP/site/maniplan/_kernels/"_compiled*.so > /dev/null   # the stock build compiled the kernel backend
"$PY" -m compileall -q -b "$TMP/site/maniplan"
find "$TMP/site/maniplan" \( -name "*.py" -o -name "*.pyx" -o -name "*.c" \) -delete
# .pyc files do not travel to the GPU box with gpurun's snapshot: keep the
# bytecode under a suffix of its own (tests/refpkg.py registers a sourceless
# loader for it, for oracle/_ref only)
find "$TMP/site/maniplan" -name '*.pyc' -exec sh -c 'mv "$1" "${1%.pyc}.refpyc"' _ {} \;
find "$TMP/site/maniplan" -name '__pycache__' -prune -exec rm -rf {} +
rm -rf "$OUT"
mkdir -p "$OUT"
cp -r "$TMP/site/maniplan" "$OUT/maniplan"
echo "reference (stock pip build, $(cd "$OUT" && find maniplan -name '*.so' | wc -l) extension module) installed into $OUT"
