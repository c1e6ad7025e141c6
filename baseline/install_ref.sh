#!/usr/bin/env bash
# Installs the UNMODIFIED reference package (`rsr`, pure Python + numpy) into
# baseline/_ref for bench.py's CPU legs (`--impl reference` and the
# cpu_baseline of the default line).  baseline/_ref is git-ignored but travels
# to the GPU box with the gpurun snapshot; /root/reference exists only in the
# build container.  The build writes into its source tree, so it runs from a
# copy under /tmp.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -f "$SRC/pyproject.toml" ] || { echo "reference source not found at $SRC" >&2; exit 1; }
TMP="$(mktemp -d /tmp/rsr_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC"/. "$TMP"/
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP" >/dev/null
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import rsr; print('reference installed:', rsr.__version__, rsr.__file__)"
