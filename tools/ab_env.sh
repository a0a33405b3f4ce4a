#!/bin/bash
# A/B a runtime variant switch: tools/ab_env.sh TAG VAR "v1 v2 ..." [bench args]
# e.g. tools/ab_env.sh wide NULPA_WIDE_MODE "0 1 2" --steps 5 --e2e-steps 0 --no-cpu-baseline
TAG=$1; VAR=$2; VALS=$3; shift 3
mkdir -p gpurun_out
for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --warmup 3 "$@" 2>&1 | tail -1 > gpurun_out/ab_${TAG}_$(basename $v).json
  python - "$TAG" "$v" <<'PY'
import json, os, sys
t, v = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"gpurun_out/ab_{t}_{os.path.basename(v)}.json"))
    names = d["config"]["tier_names"]
    tiers = " ".join(f"{n}={x:.2f}" for n, x in zip(names, d["config"]["tier_ms_per_step"]) if x)
    print(f"{t}={v}: {d['value']/1e9:.2f} G/s loop {1e3*d['config']['loop_seconds_per_step']:.2f} ms iters {d['config']['iterations']} Q {d['config']['modularity']:.3g} | {tiers}")
except Exception as e:
    print(f"{t}={v}: failed {e}")
PY
done
