#!/usr/bin/env bash
# Builds the UNMODIFIED reference (voltseg, Python + Cython) into oracle/_ref/
# with its own setup.py flags (-O3 -march=native -ffast-math -funroll-loops).
# Test/bench infrastructure only: oracle/_ref is git-ignored (never committed)
# but travels to the GPU box with gpurun, where bench.py --impl reference and
# the CPU baseline import it.  /root/reference is read-only, so the build runs
# from a scratch copy under /tmp.  Dependencies scikit-image / tifffile /
# pillow are absent (no network): --no-deps, and oracle/ref_stubs provides
# import-only stand-ins for the two modules imported at module top level.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
if [ ! -d "$SRC" ]; then echo "reference not present at $SRC; keeping prebuilt oracle/_ref" >&2; exit 0; fi
TMP="$(mktemp -d /tmp/voltseg_ref.XXXXXX)"
cp -r "$SRC"/. "$TMP"/
chmod -R u+w "$TMP"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP"
rm -rf "$TMP"
echo "built $HERE/_ref"
