mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_async_protocol_gpu.py tests/test_dist_gloo.py -x -q > gpurun_out/r2d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_pytest.log
bash tools/ab_env.sh wide NULPA_WIDE_MODE "0 1 2" --steps 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2d_ab.txt 2>&1
bash tools/ab_env.sh pipe NULPA_TEAM_PIPE "0 1" --steps 5 --e2e-steps 0 --no-cpu-baseline >> gpurun_out/r2d_ab.txt 2>&1
