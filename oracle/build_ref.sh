#!/usr/bin/env bash
# Build / install the reference itself under oracle/_ref/ (git-ignored; it
# travels to the GPU box with the gpurun snapshot).  Test infrastructure only:
# everything here is the CPU checker and the CPU baseline, never the product
# path.  Nothing from /root/reference is committed to the repo.
#
#   oracle/_ref/_kernels*.so   the reference's compiled traversal kernels
#                              (/root/reference/pkg/src/tetray/_kernels.pyx) as
#                              a standalone module, reference flags
#                              (-O3 -ffp-contract=off, pkg/setup.py:17-20)
#   oracle/_ref/site/tetray/   the unmodified reference package, installed with
#                              pip --target from a /tmp copy (its build writes
#                              into the source tree); its own _kernels
#                              extension included -- drives the drop-in tests
#                              (tetray.batch.* with kernels=our module) and the
#                              bench's reference arm
#   oracle/_ref/pkg/{tests,data,tools}
#                              the reference's own test suite and fixtures, run
#                              unmodified against the CUDA module by
#                              tests/test_reference_dropin.py
#   oracle/_ref/scenes/*.npz   the config-2 scene built by the reference's own
#                              pipeline (oracle/make_ref_scene.py), loaded by
#                              bench.py --impl reference via tetray.cli.load_compact
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${TETRAY_REF_PKG:-/root/reference/pkg}"
SRC="$REF/src/tetray/_kernels.pyx"
OUT="$HERE/_ref"
PY="${PYTHON:-python}"
if [ ! -f "$SRC" ]; then
  echo "reference source $SRC not present; skipping oracle/_ref build" >&2
  exit 0
fi
mkdir -p "$OUT/build"

# 1. standalone compiled kernels (module name `_kernels`)
SUFFIX="$("$PY" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
if [ ! -f "$OUT/_kernels$SUFFIX" ] || [ "$SRC" -nt "$OUT/_kernels$SUFFIX" ]; then
  cp "$SRC" "$OUT/build/_kernels.pyx"
  "$PY" -m cython -3 "$OUT/build/_kernels.pyx" -o "$OUT/build/_kernels.c" >/dev/null
  INC="$("$PY" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
  gcc -O3 -ffp-contract=off -fPIC -shared -I"$INC" "$OUT/build/_kernels.c" -o "$OUT/_kernels$SUFFIX"
  rm -f "$OUT/build/_kernels.pyx"
  echo "built $OUT/_kernels$SUFFIX"
fi

# 2. the reference package, installed unmodified (pip --target, offline)
if [ ! -f "$OUT/site/.installed" ]; then
  TMP="$(mktemp -d /tmp/tetray_ref.XXXXXX)"
  cp -r "$REF" "$TMP/pkg"
  rm -rf "$OUT/site"
  "$PY" -m pip install --quiet --no-index --no-build-isolation --no-deps \
      --find-links /opt/wheelhouse --target "$OUT/site" "$TMP/pkg"
  rm -rf "$TMP"
  PYTHONPATH="$OUT/site" "$PY" -c 'from tetray import backend; assert backend.active_backend() == "compiled", backend.active_backend()'
  touch "$OUT/site/.installed"
  echo "installed the reference package into $OUT/site"
fi

# 3. its own test suite + fixtures (run against the CUDA module on the GPU box)
if [ ! -f "$OUT/pkg/.copied" ]; then
  rm -rf "$OUT/pkg"
  mkdir -p "$OUT/pkg"
  cp -r "$REF/tests" "$REF/data" "$REF/tools" "$OUT/pkg/"
  touch "$OUT/pkg/.copied"
fi

# 4. the config-2 scene from the reference pipeline (minutes, once)
if [ "${TETB200_SKIP_REF_SCENE:-0}" = "0" ]; then
  PYTHONPATH="$OUT/site" "$PY" "$HERE/make_ref_scene.py" --grid 55 --layout tet20 --scheme hilbert
fi
