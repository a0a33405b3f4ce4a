# ncu --set full with source-level attribution for the tier kernels of one R27 run (pass 1)
# usage: tools/gpu/gpu_prof_src.sh TAG
TAG=${1:-src}
mkdir -p gpurun_out
prof() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"$2" -s $3 -c 1 -o gpurun_out/${TAG}_$1 python tools/profile_run.py 27 0 1 > gpurun_out/${TAG}_$1.log 2>&1
}
prof wide "k_wide" 1
prof team32 "k_team.*\(int\)32, \(int\)512, \(int\)256, \(int\)1>" 0
prof team128 "k_team.*\(int\)128, \(int\)2048, \(int\)1024, \(int\)1>" 0
prof cta512 "k_team.*\(int\)512, \(int\)8192, \(int\)6144, \(int\)1>" 0
prof thread "k_thread" 1
prof warp "k_group.*\(int\)32, \(int\)1>" 1
