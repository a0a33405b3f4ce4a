mkdir -p gpurun_out
bash tools/gpu/gpu_prof_src.sh r2p
for k in wide team32 team128 cta512 thread warp; do
  python tools/ncu_lines.py gpurun_out/r2p_$k.ncu-rep 40 > gpurun_out/r2p_lines_$k.txt 2>&1
  ncu -i gpurun_out/r2p_$k.ncu-rep --page raw --csv > gpurun_out/r2p_raw_$k.csv 2>/dev/null
done
rm -f gpurun_out/r2p_*.ncu-rep
