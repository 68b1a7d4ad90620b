#!/usr/bin/env bash
# Build the reference planner (maniplan) into oracle/_ref/ as compiled
# extension modules, from its own sources under /root/reference (read-only;
# scratch in a temp dir).  TEST / BASELINE INFRASTRUCTURE ONLY: the product
# never imports it.  The kernel backend (_compiled.pyx) gets the reference's
# own flags (pkg/setup.py:45-53); the pure-Python modules are cythonized as-is
# so the package is importable on the GPU box, where /root/reference is absent.
set -euo pipefail
REF=${REF:-/root/reference/pkg/src/maniplan}
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
OUT="$HERE/_ref"
PY=${PYTHON:-python3}
[ -d "$REF" ] || { echo "reference sources not found at $REF" >&2; exit 1; }
TMP=$(mktemp -d /tmp/cprrtc_refbuild.XXXXXX)
trap 'rm -rf "$TMP"' EXIT
mkdir -p "$TMP/src"
cp -r "$REF" "$TMP/src/maniplan"
find "$TMP/src" -name '__pycache__' -prune -exec rm -rf {} +
cat > "$TMP/setup_ref.py" <<'PYEOF'
import glob, os
from setuptools import setup, Extension
from Cython.Build import cythonize
flags = ["-O3", "-ffp-contract=off", "-fno-builtin-sin", "-fno-builtin-cos"]
kern = [Extension("maniplan._kernels._compiled", ["src/maniplan/_kernels/_compiled.pyx"],
                 extra_compile_args=flags)]
mods = []
for path in sorted(glob.glob("src/maniplan/**/*.py", recursive=True)):
    mod = path[len("src/"):-3].replace(os.sep, ".")
    mods.append(Extension(mod, [path], extra_compile_args=flags))
# the kernel backend keeps the reference's own directives (pkg/setup.py:55-60);
# the pure-Python modules keep Python semantics (bounds / negative indices / %)
exts = cythonize(kern, compiler_directives={"language_level": "3", "boundscheck": False,
                 "wraparound": False, "cdivision": True}, quiet=True, nthreads=8)
exts += cythonize(mods, compiler_directives={"language_level": "3", "binding": True},
                  quiet=True, nthreads=8)
setup(name="maniplan_ref", ext_modules=exts,
      script_args=["build_ext", "--build-lib", "build_out", "--parallel", "8"])
PYEOF
( cd "$TMP" && "$PY" setup_ref.py > build.log 2>&1 ) || { tail -30 "$TMP/build.log"; exit 1; }
rm -rf "$OUT"
mkdir -p "$OUT"
( cd "$TMP/build_out" && find maniplan -name '*.so' -print0 | while IFS= read -r -d '' f; do
      mkdir -p "$OUT/$(dirname "$f")"; cp "$f" "$OUT/$f"; done )
echo "reference built into $OUT"
