mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_pytest.log
bash tools/ab_env.sh tq NULPA_THREAD_Q "0 1" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2r_ab.txt 2>&1
bash tools/ab_env.sh tqweb NULPA_THREAD_Q "0 1" --workload web --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2r_ab.txt 2>&1
bash tools/ab_env.sh tqsbm NULPA_THREAD_Q "0 1" --workload sbm --steps 20 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2r_ab.txt 2>&1
