#!/bin/bash
# One bench line per BASELINE.json config shape (single B200), then the default headline run.
set -x
for w in sbm grid web; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --e2e-steps 1 2>&1 | tail -1 > gpurun_out/bench_$w.json
done
timeout 900 python bench.py --scale 24 --steps 3 --warmup 3 --e2e-steps 1 2>&1 | tail -1 > gpurun_out/bench_rmat24.json
timeout 1200 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_reference.json
