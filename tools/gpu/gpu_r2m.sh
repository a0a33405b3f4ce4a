mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_pytest.log
bash tools/ab_env.sh sbm NULPA_LIB "paper_2411_11468_b200/libnulpa.so" --workload sbm --steps 20 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2m_ab.txt 2>&1
bash tools/ab_env.sh r27lib NULPA_LIB "paper_2411_11468_b200/libnulpa.so paper_2411_11468_b200/var/libnulpa_vec.so" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2m_ab.txt 2>&1
bash tools/ab_env.sh l2 NULPA_L2_PERSIST "20 40 80" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2m_ab.txt 2>&1
bash tools/ab_env.sh tma NULPA_WIDE_MODE "1 2" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2m_ab.txt 2>&1
