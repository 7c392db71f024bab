#!/usr/bin/env bash
# Install the UNMODIFIED reference package `kcycle` (/root/reference/pkg) into
# the git-ignored baseline/_ref, the one offline install the task allows.
# The build writes egg-info next to the sources, and /root/reference is
# read-only, so it installs from a copy under /tmp.  Only needed in the build
# container: baseline/_ref is git-ignored but not gpurun-ignored, so it
# travels to the GPU box with the snapshot (bench.py --impl reference and
# tests/test_gpu_reference_dropin.py import it from there).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC here (GPU box?): nothing to install" >&2; exit 0; }
TMP="$(mktemp -d /tmp/kcycle_src.XXXXXX)"
cp -r "$SRC"/. "$TMP"/
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP"
rm -rf "$TMP"
# the reference's own test modules, run unchanged against CudaGridState by
# tests/test_gpu_reference_dropin.py (through the tests/refshim.py plugin)
cp -r "$SRC/tests" "$ROOT/baseline/_ref/kcycle_tests"
find "$ROOT/baseline/_ref" -name __pycache__ -prune -exec rm -rf {} +
python - <<PY
import sys; sys.path.insert(0, "$ROOT/baseline/_ref")
import kcycle, os
print("installed kcycle", kcycle.__version__, "from", os.path.dirname(kcycle.__file__))
PY
