#!/usr/bin/env bash
# Build the UNMODIFIED reference package (gemmforge, /root/reference/pkg) into
# oracle/_ref/ -- the reference arm of bench.py (`--impl reference`) and the
# strongest parity pin.  Outputs only into oracle/_ref/ (git-ignored, but it
# travels to the GPU box with the gpurun snapshot).  The build runs from a
# scratch copy under /tmp because /root/reference is read-only and setuptools
# writes build artefacts next to the sources.  No reference source is copied
# into the repository's history.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REFERENCE_ROOT:-/root/reference}/pkg"
if [ ! -d "$REF" ]; then
  echo "reference not present at $REF; skipping oracle/_ref build" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/gemmforge_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"
chmod -R u+w "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import gemmforge
from gemmforge.backends import available_backends
assert "c" in available_backends(), "compiled backend did not build"
print("oracle/_ref: gemmforge", gemmforge.__version__, "backends", available_backends())
PY
