#!/bin/bash
# One GPU round-trip: parity tests, smoke, default bench, launch list, one ncu --set full capture.
# usage: tools/gpu_check.sh TAG
TAG=${1:-chk}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json
