#!/bin/bash
# The reference's own test suite (pkg/tests, copied from /root/reference into
# the git-ignored scratch_reftests/ in the build container -- never committed)
# against the B200 engine through the drop-in package dropin/permanent.
#   bash tools/run_reference_suite.sh OUT.txt [pytest args]
set -u
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
OUT="$(realpath -m "${1:-$ROOT/gpurun_out/refsuite.txt}")"
if [ ! -d "$ROOT/scratch_reftests" ]; then
  if [ -d /root/reference/pkg/tests ]; then
    cp -r /root/reference/pkg/tests "$ROOT/scratch_reftests"
  else
    echo "no scratch_reftests/ (copy /root/reference/pkg/tests there first)" > "$OUT"; exit 0
  fi
fi
cd "$ROOT/scratch_reftests" && PYTHONPATH="$ROOT/dropin" NUMBA_CACHE_DIR=/tmp/numba_cache \
  python -m pytest -q -p no:cacheprovider -rA "${@:2}" > "$OUT" 2>&1
echo "exit $?" >> "$OUT"
