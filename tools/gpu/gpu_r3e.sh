mkdir -p gpurun_out
bash tools/ab_env.sh r27 NULPA_LIB "paper_2411_11468_b200/libnulpa.so paper_2411_11468_b200/var/libnulpa_mid4096.so" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r3e_ab.txt 2>&1
bash tools/ab_env.sh web NULPA_LIB "paper_2411_11468_b200/libnulpa.so paper_2411_11468_b200/var/libnulpa_mid4096.so" --workload web --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r3e_ab.txt 2>&1
