#!/bin/bash
# Grid quality and loop time per NULPA_MIN_CHUNK variant.
for F in "$@"; do
  echo "== variant: $F"
  NULPA_NVCC_FLAGS="$F" python -c "from paper_2411_11468_b200 import build as b; b.build_library(force=True)" || continue
  python tools/grid_quality.py 2>&1 | grep "schedule 4"
  python bench.py --workload grid --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('grid4096 bench', round(d['value']/1e9,2), 'G/s loop', round(d['config']['loop_seconds_per_step']*1e3,1), 'ms iters', d['config']['iterations'], 'Q', round(d['config']['modularity'],4))"
done
