mkdir -p gpurun_out
bash tools/ab_env.sh grid NULPA_WARP_CHUNKS "0 1" --workload grid --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r3a_ab.txt 2>&1
NULPA_WARP_CHUNKS=1 timeout 600 python -m pytest tests -m gpu -q -k "lattice or grid" > gpurun_out/r3a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_pytest.log
