#!/bin/bash
# Rebuild with extra nvcc flags and time one R-MAT run per variant.
# usage: tools/variant_bench.sh SCALE "FLAGS1" "FLAGS2" ...
SCALE=$1; shift
for F in "$@"; do
  echo "== variant: $F"
  NULPA_NVCC_FLAGS="$F" python -c "from paper_2411_11468_b200 import build as b; b.build_library(force=True)" || continue
  python tools/tier_bench.py $SCALE 3 iters=1 2>&1 | tail -3 | head -2
  python tools/tier_bench.py $SCALE 3 2>&1 | tail -3 | head -2
done
