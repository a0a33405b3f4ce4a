mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2z_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2z_bench.json
