#!/bin/bash
# GPU round trip: tests, smoke, bench lines for every workload, launch list, ncu capture.
# usage: tools/gpu_full.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
bash tools/gpu_check.sh $TAG
for w in sbm grid web; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --e2e-steps 1 2>&1 | tail -1 > gpurun_out/${TAG}_bench_$w.json
done
timeout 900 python bench.py --scale 24 --steps 3 --warmup 3 --e2e-steps 1 2>&1 | tail -1 > gpurun_out/${TAG}_bench_rmat24.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_launches_bench.log 2>&1
timeout 1200 bash tools/profile_kernels.sh 27 ${TAG}_r27_full 0 6 > gpurun_out/${TAG}_ncu_full.log 2>&1
# every tier kernel of one run (3 passes): DRAM bytes per launch for bench.py's roofline.traffic
timeout 1500 ncu --set full --clock-control none -k regex:"k_(thread|group|team|wide|cluster|hub_accum)" -c 40 \
  -o gpurun_out/${TAG}_r27_tiers python tools/profile_run.py 27 0 1 > gpurun_out/${TAG}_ncu_tiers.log 2>&1
python tools/ncu_traffic.py gpurun_out/${TAG}_r27_tiers.ncu-rep > gpurun_out/${TAG}_ncu_traffic_r27.json 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_r27_full.ncu-rep gpurun_out/${TAG}_r27_tiers.ncu-rep > gpurun_out/${TAG}_ncu_summary.txt 2>&1
rm -f gpurun_out/${TAG}_r27_tiers.ncu-rep   # (the result directory comes back only under 64 MiB)
