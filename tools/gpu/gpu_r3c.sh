mkdir -p gpurun_out
bash tools/ab_env.sh grid NULPA_CHUNK_PIPE "0 1" --workload grid --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r3c_ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "lattice or grid or invariant or kat or async" > gpurun_out/r3c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_pytest.log
