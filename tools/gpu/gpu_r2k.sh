mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_pytest.log
bash tools/ab_env.sh r27lib NULPA_LIB "paper_2411_11468_b200/libnulpa.so paper_2411_11468_b200/var/libnulpa_wide512.so paper_2411_11468_b200/var/libnulpa_w512tpf.so" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2k_ab.txt 2>&1
bash tools/ab_env.sh sbmlib NULPA_LIB "paper_2411_11468_b200/libnulpa.so paper_2411_11468_b200/var/libnulpa_w512tpf.so" --workload sbm --steps 20 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2k_ab.txt 2>&1
bash tools/ab_env.sh weblib NULPA_LIB "paper_2411_11468_b200/libnulpa.so paper_2411_11468_b200/var/libnulpa_w512tpf.so" --workload web --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2k_ab.txt 2>&1
bash tools/gpu/gpu_prof_src.sh r2k
