#!/usr/bin/env bash
# Install the UNMODIFIED reference package (superlse, pure Python) into
# baseline/_ref for bench.py's reference arm and cpu_baseline legs.
# /root/reference is read-only and its pyproject.toml sits in pkg/, so the
# install runs from a copy under /tmp.  numpy/scipy are already in the image
# (--no-deps).  baseline/_ref is git-ignored but travels to the GPU box with
# the gpurun snapshot.
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference}"
TMP="$(mktemp -d /tmp/superlse_ref.XXXXXX)"
cp -r "$SRC/pkg/." "$TMP/"
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$REPO/baseline/_ref" "$TMP"
rm -rf "$TMP"
PYTHONPATH="$REPO/baseline/_ref" python -c "import superlse; print('installed', superlse.__file__)"
