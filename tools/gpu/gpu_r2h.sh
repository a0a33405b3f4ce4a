mkdir -p gpurun_out
timeout 300 python tools/experiments/dist_debug.py 14 sync > gpurun_out/r2h_dist.log 2>&1
bash tools/ab_env.sh sbmgrp NULPA_GROUP_STEPS "1 8" --workload sbm --steps 20 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2h_ab.txt 2>&1
bash tools/ab_env.sh sbmpair NULPA_THREAD_PAIR "0 1" --workload sbm --steps 20 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2h_ab.txt 2>&1
bash tools/ab_env.sh sbmbatch NULPA_BATCH_PASSES "1 4" --workload sbm --steps 20 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2h_ab.txt 2>&1
bash tools/ab_env.sh r27grp NULPA_GROUP_STEPS "1 8" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2h_ab.txt 2>&1
bash tools/ab_env.sh r27lib NULPA_LIB "paper_2411_11468_b200/libnulpa.so paper_2411_11468_b200/var/libnulpa_minb5.so" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2h_ab.txt 2>&1
timeout 1500 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --dropin-steps 1 > gpurun_out/r2h_bench.log 2> gpurun_out/r2h_bench.err; tail -1 gpurun_out/r2h_bench.log > gpurun_out/r2h_bench.json
free -g > gpurun_out/r2h_host.txt; nproc >> gpurun_out/r2h_host.txt; df -h /dev/shm >> gpurun_out/r2h_host.txt
