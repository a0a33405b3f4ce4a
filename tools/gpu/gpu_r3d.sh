mkdir -p gpurun_out/r3d
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3d/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r3d/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3d/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3d/smoke.log
timeout 1200 python bench.py > gpurun_out/r3d/bench.log 2> gpurun_out/r3d/bench.err; tail -1 gpurun_out/r3d/bench.log > gpurun_out/r3d/bench.json
