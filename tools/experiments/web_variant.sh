#!/bin/bash
# Web-like bench (loop time and tier split) per nvcc-flag variant.
for F in "$@"; do
  echo "== variant: $F"
  NULPA_NVCC_FLAGS="$F" python -c "from paper_2411_11468_b200 import build as b; b.build_library(force=True)" || continue
  python bench.py --workload web --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); c=d['config']; print('web', round(d['value']/1e9,2), 'G/s loop', round(c['loop_seconds_per_step']*1e3,1), [(n, round(t,2)) for n,t in zip(c['tier_names'], c['tier_ms_per_step']) if t])"
done
