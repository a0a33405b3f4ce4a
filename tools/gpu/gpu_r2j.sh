mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_pytest.log
bash tools/ab_env.sh r27lib NULPA_LIB "paper_2411_11468_b200/libnulpa.so paper_2411_11468_b200/var/libnulpa_wide512.so" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2j_ab.txt 2>&1
bash tools/ab_env.sh r27tg NULPA_THREAD_GROUP "1" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2j_ab.txt 2>&1
bash tools/ab_env.sh sbm NULPA_THREAD_GROUP "0 1" --workload sbm --steps 20 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2j_ab.txt 2>&1
bash tools/gpu/gpu_prof_src.sh r2j
timeout 1200 python bench.py > gpurun_out/r2j_bench.log 2> gpurun_out/r2j_bench.err; tail -1 gpurun_out/r2j_bench.log > gpurun_out/r2j_bench.json
