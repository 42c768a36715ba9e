#!/usr/bin/env bash
# Build the reference package (hybridcolor, /root/reference/pkg) with its own
# compiled Cython/OpenMP kernel backend into oracle/_ref/ (git-ignored; it
# travels to the GPU box with the gpurun snapshot).  The reference tree is
# read-only, so the pip build runs from a scratch copy under /tmp.  The
# default gcc in this image lacks libgomp.spec, hence CC=/usr/bin/gcc.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
if [ ! -d "$SRC" ]; then
  echo "reference tree $SRC not present; keeping existing oracle/_ref" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/hcref.XXXXXX)"
cp -r "$SRC/." "$TMP/"
rm -rf "$HERE/_ref"
( cd "$TMP" && CC=/usr/bin/gcc LDSHARED="/usr/bin/gcc -shared" \
    python -m pip install -q --no-index --no-build-isolation --no-deps \
      --find-links /opt/wheelhouse --target "$HERE/_ref" . )
rm -rf "$TMP"
# the reference's own test suite (run against the cuda backend by
# tests/test_reference_suite.py through tests/refsuite_plugin.py)
cp -r "$SRC/tests" "$HERE/_ref/tests"
python - <<PY
import sys; sys.path.insert(0, "$HERE/_ref")
import hybridcolor
assert "cython" in hybridcolor.available_backends(), hybridcolor.available_backends()
print("oracle/_ref: hybridcolor", hybridcolor.__version__, hybridcolor.available_backends())
PY
