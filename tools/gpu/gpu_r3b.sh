mkdir -p gpurun_out
bash tools/ab_env.sh grid NULPA_WARP_CHUNKS "0" --workload grid --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r3b_ab.txt 2>&1
