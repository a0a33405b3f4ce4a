mkdir -p gpurun_out
bash tools/ab_env.sh wmode NULPA_WIDE_MODE "0 1 3" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2q_ab.txt 2>&1
bash tools/ab_env.sh dedup NULPA_DEDUP_LATER "0 1" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2q_ab.txt 2>&1
bash tools/ab_env.sh wmodeweb NULPA_WIDE_MODE "0 3" --workload web --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2q_ab.txt 2>&1
