mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "modularity or quality or stats or dist or smoke" > gpurun_out/r2t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2t_bench.json
timeout 600 python bench.py --workload web --steps 3 --warmup 3 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2t_bench_web.json
