# ncu --set full with source-level attribution for the dominant tier kernels of one R27 run
# usage: tools/gpu/gpu_prof_src.sh TAG [LIB]
TAG=${1:-src}
mkdir -p gpurun_out
[ -n "$2" ] && export NULPA_LIB=$2
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_wide" -s 1 -c 1 -o gpurun_out/${TAG}_wide python tools/profile_run.py 27 0 1 > gpurun_out/${TAG}_wide.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_team.*\(int\)32, \(int\)512, \(int\)256, \(int\)1>" -s 0 -c 1 -o gpurun_out/${TAG}_team32 python tools/profile_run.py 27 0 1 > gpurun_out/${TAG}_team32.log 2>&1
