mkdir -p gpurun_out
bash tools/gpu/gpu_prof_src.sh r2p
