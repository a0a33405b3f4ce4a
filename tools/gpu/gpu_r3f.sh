mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "cached_plan or sync_step_vs_port" > gpurun_out/r3f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_pytest.log
