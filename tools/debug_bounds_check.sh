#!/bin/bash
# The GPU parity suite against the bounds-assert build:
# every PERM_CHECK in the kernels (csrc/common.cuh) traps on a violated
# index bound, so a passing run is the memory-safety evidence that
# compute-sanitizer (closed on this GPU pool) would otherwise give.
#   make -C paper_2510_03421_b200/csrc debug      # here (CPU), ~3.5 min
#   bash tools/debug_bounds_check.sh OUT.txt      # on the GPU box
set -u
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
OUT="$(realpath -m "${1:-$ROOT/gpurun_out/debug_bounds.txt}")"
LIB="$ROOT/paper_2510_03421_b200/libpermanent_b200_debug.so"
if [ ! -f "$LIB" ]; then echo "no $LIB (make -C paper_2510_03421_b200/csrc debug)" > "$OUT"; exit 0; fi
cd "$ROOT" && PERMANENT_B200_LIB="$LIB" python -m pytest tests -m gpu -q -p no:cacheprovider \
  --deselect tests/test_gpu_acceptance.py::test_criterion_07_dispatch_within_125x > "$OUT" 2>&1
echo "exit $?" >> "$OUT"
