#!/usr/bin/env bash
# Build the reference's own compiled traversal kernels (tetray._kernels,
# /root/reference/pkg/src/tetray/_kernels.pyx) into oracle/_ref/ as a
# standalone extension module `_kernels`, with the reference's own flags
# (-O3 -ffp-contract=off, pkg/setup.py:17-20).  Test infrastructure only:
# the oracle/_ref module is the CPU checker and the CPU baseline, never the
# product path.  Nothing from /root/reference is copied into the repo: the
# Cython-generated C and the .so live only under oracle/_ref/ (git-ignored).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${TETRAY_REF_PYX:-/root/reference/pkg/src/tetray/_kernels.pyx}"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "reference source $SRC not present; skipping oracle/_ref build" >&2
  exit 0
fi
mkdir -p "$OUT/build"
PY="${PYTHON:-python}"
# Cythonize under a stand-alone module name so the .so imports as `_kernels`.
cp "$SRC" "$OUT/build/_kernels.pyx"
"$PY" -m cython -3 "$OUT/build/_kernels.pyx" -o "$OUT/build/_kernels.c" >/dev/null
SUFFIX="$("$PY" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
INC="$("$PY" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
gcc -O3 -ffp-contract=off -fPIC -shared -I"$INC" "$OUT/build/_kernels.c" -o "$OUT/_kernels$SUFFIX"
rm -f "$OUT/build/_kernels.pyx"
echo "built $OUT/_kernels$SUFFIX"
