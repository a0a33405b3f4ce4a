mkdir -p gpurun_out
timeout 300 python tools/experiments/dist_debug.py 14 sync > gpurun_out/r2i_dist.log 2>&1
timeout 600 python tools/experiments/hang_repro.py > gpurun_out/r2i_hang.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_hang.log
bash tools/ab_env.sh r27lib NULPA_LIB "paper_2411_11468_b200/var/libnulpa_nofence.so paper_2411_11468_b200/var/libnulpa_skip.so paper_2411_11468_b200/var/libnulpa_adapt.so" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/r2i_ab.txt 2>&1
bash tools/ab_env.sh r27pair NULPA_THREAD_PAIR "0 1" --steps 5 --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline >> gpurun_out/r2i_ab.txt 2>&1
bash tools/gpu/gpu_prof_src.sh r2i
